"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two libraries, both checkers, never the product:
  * ``Oracle``  -> oracle/_build/liboracle.so, the C restatement (mhw_oracle.c);
  * ``RefLib``  -> oracle/_ref/libmhwalk_ref.so, the unmodified reference
    sources compiled in place (oracle/Makefile) plus oracle/ref_driver.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmhwalk_ref.so")
REFERENCE_TREE = "/root/reference/proj"

DEEPWALK, NODE2VEC, METAPATH2VEC, EDGE2VEC, FAIRWALK = range(5)
MODEL_NAMES = ["deepwalk", "node2vec", "metapath2vec", "edge2vec", "fairwalk"]
INIT_RANDOM, INIT_HIGH_WEIGHT, INIT_BURN_IN = range(3)
RNG_XOSHIRO, RNG_PHILOX = 0, 1
SAMPLER_MH, SAMPLER_ALIAS, SAMPLER_DIRECT, SAMPLER_REJECTION = range(4)
ORDER_WALKER, ORDER_STEP = 0, 1
NO_AFFIX = 0xFFFFFFFF

_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)


def _ptr(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def build(ref: bool | None = None) -> None:
    """Compile the oracle (and the reference, when its tree is present)."""
    target = "all" if ref is None else ("ref" if ref else "oracle")
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


class _OgGraph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("offsets", _u64p), ("nbr", _u32p),
                ("w", _dp), ("ntype", _u16p), ("etype", _u16p), ("n_ntypes", C.c_uint16),
                ("n_etypes", C.c_uint16), ("symmetric", C.c_int)]


class _OgModel(C.Structure):
    _fields_ = [("kind", C.c_int), ("p", C.c_double), ("q", C.c_double), ("metapath", _u16p),
                ("mp_len", C.c_uint32), ("M", _dp), ("M_dim", C.c_uint32),
                ("type_counts", _u32p), ("num_types", C.c_uint16)]


class _OgConfig(C.Structure):
    _fields_ = [("K", C.c_uint32), ("L", C.c_uint32), ("seed", C.c_uint64), ("init_kind", C.c_int),
                ("burn_in_steps", C.c_uint32), ("hw_sample_size", C.c_uint32), ("rng", C.c_int),
                ("order", C.c_int), ("replica_degree", C.c_uint32), ("sampler", C.c_int), ("proposal", C.c_int)]


class _OgStats(C.Structure):
    _fields_ = [("walks", C.c_uint64), ("early", C.c_uint64), ("skipped", C.c_uint64),
                ("steps", C.c_uint64), ("init_calls", C.c_uint64), ("trials", C.c_uint64)]


@dataclass
class HostGraph:
    """CSR in the reference's host layout (graph.hpp:15-55): u64 offsets,
    u32 sorted ids, f64 weights, optional u16 node/edge types."""
    offsets: np.ndarray
    nbr: np.ndarray
    w: np.ndarray
    ntype: np.ndarray | None = None
    etype: np.ndarray | None = None
    n_ntypes: int = 0
    n_etypes: int = 0
    symmetric: bool = True

    def __post_init__(self):
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.uint64)
        self.nbr = np.ascontiguousarray(self.nbr, dtype=np.uint32)
        self.w = np.ascontiguousarray(self.w, dtype=np.float64)
        if self.ntype is not None:
            self.ntype = np.ascontiguousarray(self.ntype, dtype=np.uint16)
        if self.etype is not None:
            self.etype = np.ascontiguousarray(self.etype, dtype=np.uint16)

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    @property
    def m(self) -> int:
        return len(self.nbr)

    def degree(self, v):
        return int(self.offsets[v + 1] - self.offsets[v])

    def neighbors_of(self, v):
        return self.nbr[self.offsets[v]:self.offsets[v + 1]]

    def weights_of(self, v):
        return self.w[self.offsets[v]:self.offsets[v + 1]]

    def struct(self) -> _OgGraph:
        s = _OgGraph()
        s.n, s.m = self.n, self.m
        s.offsets, s.nbr, s.w = _ptr(self.offsets, _u64p), _ptr(self.nbr, _u32p), _ptr(self.w, _dp)
        s.ntype, s.etype = _ptr(self.ntype, _u16p), _ptr(self.etype, _u16p)
        s.n_ntypes, s.n_etypes, s.symmetric = self.n_ntypes, self.n_etypes, int(self.symmetric)
        return s


@dataclass
class ModelDesc:
    """Walk model parameters (models.hpp:40-47)."""
    kind: int = DEEPWALK
    p: float = 1.0
    q: float = 1.0
    metapath: list = field(default_factory=list)
    type_matrix: np.ndarray | None = None  # dim x dim


@dataclass
class WalkCfg:
    """WalkConfig + InitStrategy (engine.hpp:19-26, samplers.hpp:29-34)."""
    K: int = 10
    L: int = 80
    seed: int = 0
    init_kind: int = INIT_RANDOM
    burn_in_steps: int = 100
    hw_sample_size: int = 32
    # engine chain layout: hub replicas for node-keyed models (0 = 256);
    # NO_REPLICAS = one chain per state, the reference's SamplerManager
    replica_degree: int = 0xFFFFFFFF
    # SamplerKind (engine.hpp:14): 0 mh, 1 alias, 2 direct, 3 rejection
    sampler: int = 0
    # M-H proposal (engine extension): 0 uniform (mh_transition), 1 static-weight alias + Hastings
    proposal: int = 0


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    """The C restatement (mhw_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.lib = L
        L.og_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.og_philox_key.argtypes = [C.c_uint64, C.c_uint32, _u32p]
        L.og_xoshiro_walker_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                              C.c_uint32, _u32p]
        L.og_build_csr.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.c_int, C.c_uint32,
                                   _u32p, _u64p, C.POINTER(_u64p), C.POINTER(_u32p), C.POINTER(_dp)]
        L.og_rmat_pairs.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                    C.c_uint64, _u64p, C.POINTER(_u32p), C.POINTER(_u32p)]
        L.og_hetero_pairs.argtypes = [C.c_uint32, C.c_uint64, _u32p, _u32p, _u64p,
                                      C.POINTER(_u32p), C.POINTER(_u32p)]
        L.og_pair_weight.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_float, C.c_float]
        L.og_pair_weight.restype = C.c_float
        L.og_pair_etype.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.og_pair_etype.restype = C.c_uint32
        L.og_pair_weights.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, C.c_float, C.c_float, _fp]
        L.og_pair_etypes.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, C.c_uint32, _u16p]
        L.og_graph_checksum.argtypes = [C.c_uint32, _u64p, _u32p, _dp]
        L.og_graph_checksum.restype = C.c_uint64
        L.og_alias_tables.argtypes = [C.c_uint32, _u64p, _dp, _dp, _u32p]
        L.og_free.argtypes = [C.c_void_p]
        L.og_model_bind.argtypes = [C.POINTER(_OgGraph), C.POINTER(_OgModel), C.c_char_p, C.c_size_t]
        L.og_decide.argtypes = [C.POINTER(_OgGraph), C.POINTER(_OgModel), C.c_uint64, _u32p, _u32p,
                                _u32p, _u32p, _dp, _dp, _dp, _u8p]
        L.og_decide_hastings.argtypes = [C.POINTER(_OgGraph), C.POINTER(_OgModel), C.c_uint64, _u32p, _u32p,
                                         _u32p, _u32p, _dp, _dp, _dp, _u8p]
        L.og_alias_build.argtypes = [C.c_uint32, _dp, _dp, _u32p]
        L.og_check.argtypes = [C.POINTER(_OgGraph), C.POINTER(_OgModel), C.c_uint64, C.c_uint64, _u32p, _u32p,
                               C.c_uint64, _u64p, _dp]
        L.og_direct_sample_u.argtypes = [C.c_uint32, _dp, C.c_double]
        L.og_direct_sample_u.restype = C.c_uint32
        L.og_slot_count.argtypes = [C.POINTER(_OgGraph), C.POINTER(_OgModel)]
        L.og_slot_count.restype = C.c_uint64
        L.og_init_philox.argtypes = [C.POINTER(_OgGraph), C.POINTER(_OgModel), C.POINTER(_OgConfig),
                                     C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
        L.og_generate_walks.argtypes = [C.POINTER(_OgGraph), C.POINTER(_OgModel), C.POINTER(_OgConfig),
                                        C.c_uint32, _u32p, _u32p, _u64p, C.POINTER(_OgStats),
                                        C.c_char_p, C.c_size_t]
        L.og_walk_isolated.argtypes = [C.POINTER(_OgGraph), C.POINTER(_OgModel), C.POINTER(_OgConfig), C.c_uint64,
                                       _u32p, C.c_uint32, _u32p, _u32p, _u64p, C.POINTER(_OgStats), C.c_char_p,
                                       C.c_size_t]

    # ---------------------------------------------------------------- rng
    def philox(self, ctr, key):
        c = np.ascontiguousarray(ctr, dtype=np.uint32)
        k = np.ascontiguousarray(key, dtype=np.uint32)
        out = np.zeros(4, dtype=np.uint32)
        self.lib.og_philox4x32_10(_ptr(c, _u32p), _ptr(k, _u32p), _ptr(out, _u32p))
        return out

    def xoshiro_walker_draws(self, seed, node, k, bound, count):
        out = np.zeros(count, dtype=np.uint32)
        self.lib.og_xoshiro_walker_draws(seed, node, k, bound, count, _ptr(out, _u32p))
        return out

    # -------------------------------------------------------------- graphs
    def build_csr(self, src, dst, w=None, symmetrize=False, n_nodes=0) -> HostGraph:
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        wa = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        n, m = C.c_uint32(), C.c_uint64()
        po, pn, pw = _u64p(), _u32p(), _dp()
        rc = self.lib.og_build_csr(len(src), _ptr(src, _u32p), _ptr(dst, _u32p), _ptr(wa, _dp),
                                   int(symmetrize), n_nodes, C.byref(n), C.byref(m), C.byref(po),
                                   C.byref(pn), C.byref(pw))
        if rc:
            raise OracleError(rc, "build_csr failed")
        off = np.ctypeslib.as_array(po, shape=(n.value + 1,)).copy()
        nb = np.ctypeslib.as_array(pn, shape=(max(m.value, 1),))[:m.value].copy()
        ww = np.ctypeslib.as_array(pw, shape=(max(m.value, 1),))[:m.value].copy()
        for p in (po, pn, pw):
            self.lib.og_free(C.cast(p, C.c_void_p))
        return HostGraph(off, nb, ww, symmetric=bool(symmetrize))

    def _pairs(self, plo, phi, count):
        lo = np.ctypeslib.as_array(plo, shape=(max(count, 1),))[:count].copy()
        hi = np.ctypeslib.as_array(phi, shape=(max(count, 1),))[:count].copy()
        self.lib.og_free(C.cast(plo, C.c_void_p))
        self.lib.og_free(C.cast(phi, C.c_void_p))
        return lo, hi

    def rmat_pairs(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
        cnt = C.c_uint64()
        plo, phi = _u32p(), _u32p()
        rc = self.lib.og_rmat_pairs(scale, edge_factor, a, b, c, seed, C.byref(cnt), C.byref(plo),
                                    C.byref(phi))
        if rc:
            raise OracleError(rc, "rmat failed")
        return self._pairs(plo, phi, cnt.value)

    def hetero_pairs(self, n_nodes, seed=1):
        nA, nP, cnt = C.c_uint32(), C.c_uint32(), C.c_uint64()
        plo, phi = _u32p(), _u32p()
        rc = self.lib.og_hetero_pairs(n_nodes, seed, C.byref(nA), C.byref(nP), C.byref(cnt),
                                      C.byref(plo), C.byref(phi))
        if rc:
            raise OracleError(rc, "hetero failed")
        lo, hi = self._pairs(plo, phi, cnt.value)
        return lo, hi, nA.value, nP.value

    def pair_weights(self, seed, lo, hi, wlo, whi):
        lo = np.ascontiguousarray(lo, dtype=np.uint32)
        hi = np.ascontiguousarray(hi, dtype=np.uint32)
        out = np.zeros(len(lo), dtype=np.float32)
        self.lib.og_pair_weights(seed, len(lo), _ptr(lo, _u32p), _ptr(hi, _u32p), wlo, whi, _ptr(out, _fp))
        return out

    def pair_etypes(self, seed, lo, hi, n_types):
        lo = np.ascontiguousarray(lo, dtype=np.uint32)
        hi = np.ascontiguousarray(hi, dtype=np.uint32)
        out = np.zeros(len(lo), dtype=np.uint16)
        self.lib.og_pair_etypes(seed, len(lo), _ptr(lo, _u32p), _ptr(hi, _u32p), n_types, _ptr(out, _u16p))
        return out

    def graph_checksum(self, offsets, nbr, w=None):
        """graph_checksum of tools/mhwalk.cpp:107-122 (FNV-1a)."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nb = np.ascontiguousarray(nbr, dtype=np.uint32)
        wa = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        return int(self.lib.og_graph_checksum(len(off) - 1, _ptr(off, _u64p), _ptr(nb, _u32p), _ptr(wa, _dp)))

    # -------------------------------------------------------------- models
    def bind(self, g: HostGraph, md: ModelDesc):
        """Returns (og_graph struct, og_model struct, keepalive) after bind."""
        gs = g.struct()
        ms = _OgModel()
        keep = [g]
        ms.kind, ms.p, ms.q = md.kind, md.p, md.q
        if md.metapath:
            mp = np.ascontiguousarray(md.metapath, dtype=np.uint16)
            keep.append(mp)
            ms.metapath, ms.mp_len = _ptr(mp, _u16p), len(mp)
        if md.type_matrix is not None:
            M = np.ascontiguousarray(md.type_matrix, dtype=np.float64)
            keep.append(M)
            ms.M, ms.M_dim = _ptr(M, _dp), M.shape[0]
        if md.kind == FAIRWALK:
            tc = np.zeros(max(g.n * g.n_ntypes, 1), dtype=np.uint32)
            keep.append(tc)
            ms.type_counts = _ptr(tc, _u32p)
        err = C.create_string_buffer(512)
        rc = self.lib.og_model_bind(C.byref(gs), C.byref(ms), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return gs, ms, keep

    def decide(self, g, md, pos, affix, cand, last, u):
        gs, ms, keep = self.bind(g, md)
        n = len(pos)
        arrs = [np.ascontiguousarray(x, dtype=np.uint32) for x in (pos, affix, cand, last)]
        uu = np.ascontiguousarray(u, dtype=np.float64)
        wc, wl = np.zeros(n), np.zeros(n)
        acc = np.zeros(n, dtype=np.uint8)
        self.lib.og_decide(C.byref(gs), C.byref(ms), n, *[_ptr(a, _u32p) for a in arrs],
                           _ptr(uu, _dp), _ptr(wc, _dp), _ptr(wl, _dp), _ptr(acc, _u8p))
        return wc, wl, acc

    def decide_hastings(self, g, md, pos, affix, cand, last, u):
        """Alias-proposal decisions: (r_c, r_l, accept) with r = w'/w the
        model's dynamic factor and the Hastings accept of og_hastings."""
        gs, ms, keep = self.bind(g, md)
        n = len(pos)
        arrs = [np.ascontiguousarray(x, dtype=np.uint32) for x in (pos, affix, cand, last)]
        uu = np.ascontiguousarray(u, dtype=np.float64)
        rc, rl = np.zeros(n), np.zeros(n)
        acc = np.zeros(n, dtype=np.uint8)
        self.lib.og_decide_hastings(C.byref(gs), C.byref(ms), n, *[_ptr(a, _u32p) for a in arrs],
                                    _ptr(uu, _dp), _ptr(rc, _dp), _ptr(rl, _dp), _ptr(acc, _u8p))
        return rc, rl, acc

    def alias_build(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        prob = np.zeros(len(w))
        alias = np.zeros(len(w), dtype=np.uint32)
        rc = self.lib.og_alias_build(len(w), _ptr(w, _dp), _ptr(prob, _dp), _ptr(alias, _u32p))
        if rc:
            raise OracleError(rc, "alias_build: no positive weight")
        return prob, alias

    def alias_tables(self, offsets, w):
        """Static alias tables of every node (engine.cpp:136-146), CSR order."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        wa = np.ascontiguousarray(w, dtype=np.float64)
        prob = np.zeros(len(wa))
        alias = np.zeros(len(wa), dtype=np.uint32)
        self.lib.og_alias_tables(len(off) - 1, _ptr(off, _u64p), _ptr(wa, _dp), _ptr(prob, _dp), _ptr(alias, _u32p))
        return prob, alias

    def _cfg(self, cfg: WalkCfg, rng, order):
        c = _OgConfig()
        c.K, c.L, c.seed = cfg.K, cfg.L, cfg.seed
        c.init_kind, c.burn_in_steps, c.hw_sample_size = cfg.init_kind, cfg.burn_in_steps, cfg.hw_sample_size
        c.rng, c.order = rng, order
        c.replica_degree = cfg.replica_degree
        c.sampler = cfg.sampler
        c.proposal = cfg.proposal
        return c

    def generate_walks(self, g, md, cfg: WalkCfg, rng=RNG_XOSHIRO, order=ORDER_WALKER, stride=None):
        """Returns (rows uint32[n_rows, stride], lens uint32[n_rows], stats dict)."""
        gs, ms, keep = self.bind(g, md)
        c = self._cfg(cfg, rng, order)
        stride = stride or cfg.L + 1
        total = g.n * cfg.K
        rows = np.zeros((max(total, 1), stride), dtype=np.uint32)
        lens = np.zeros(max(total, 1), dtype=np.uint32)
        nrows = C.c_uint64()
        st = _OgStats()
        err = C.create_string_buffer(512)
        rc = self.lib.og_generate_walks(C.byref(gs), C.byref(ms), C.byref(c), stride,
                                        _ptr(rows, _u32p), _ptr(lens, _u32p), C.byref(nrows),
                                        C.byref(st), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        k = nrows.value
        stats = dict(walks=st.walks, early_terminations=st.early, skipped_starts=st.skipped,
                     steps=st.steps, init_calls=st.init_calls, trials=st.trials)
        return rows[:k], lens[:k], stats

    def walk_isolated(self, g, md, cfg: WalkCfg, starts, stride=None):
        """og_walk_isolated: each walker of `starts` (K per start, walker id
        v*K + k) alone with a fresh manager, Philox layout, walker-major.
        Returns (rows, lens, stats) like generate_walks."""
        gs, ms, keep = self.bind(g, md)
        c = self._cfg(cfg, RNG_PHILOX, ORDER_WALKER)
        stride = stride or cfg.L + 1
        st_ = np.ascontiguousarray(starts, dtype=np.uint32)
        total = len(st_) * cfg.K
        rows = np.zeros((max(total, 1), stride), dtype=np.uint32)
        lens = np.zeros(max(total, 1), dtype=np.uint32)
        nrows = C.c_uint64()
        st = _OgStats()
        err = C.create_string_buffer(512)
        rc = self.lib.og_walk_isolated(C.byref(gs), C.byref(ms), C.byref(c), len(st_), _ptr(st_, _u32p), stride,
                                       _ptr(rows, _u32p), _ptr(lens, _u32p), C.byref(nrows), C.byref(st), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        k = nrows.value
        stats = dict(walks=st.walks, early_terminations=st.early, skipped_starts=st.skipped,
                     steps=st.steps, init_calls=st.init_calls, trials=st.trials)
        return rows[:k], lens[:k], stats

    def check(self, g, md, seed, pos, affix, draws):
        """og_check: per-state (kl, counts) of cmd_check's chain audit."""
        gs, ms, keep = self.bind(g, md)
        pos = np.ascontiguousarray(pos, dtype=np.uint32)
        aff = np.ascontiguousarray(affix, dtype=np.uint32)
        deg = np.diff(g.offsets).astype(np.int64)[pos]
        counts = np.zeros(max(int(deg.sum()), 1), dtype=np.uint64)
        kl = np.zeros(len(pos))
        self.lib.og_check(C.byref(gs), C.byref(ms), seed, len(pos), _ptr(pos, _u32p), _ptr(aff, _u32p), draws,
                          _ptr(counts, _u64p), _ptr(kl, _dp))
        return kl, counts[:int(deg.sum())]

    def init_philox(self, g, md, cfg: WalkCfg, v, affix, slot):
        gs, ms, keep = self.bind(g, md)
        c = self._cfg(cfg, RNG_PHILOX, ORDER_STEP)
        out = C.c_uint32()
        ok = self.lib.og_init_philox(C.byref(gs), C.byref(ms), C.byref(c), v, affix, slot, C.byref(out))
        return out.value if ok else None



class RefLib:
    """The unmodified reference library (oracle/_ref/libmhwalk_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO) or os.path.isdir(REFERENCE_TREE)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_new.restype = C.c_void_p
        L.ref_graph_new.argtypes = [C.c_uint32, C.c_uint64, _u64p, _u32p, _dp, _u16p, C.c_uint16,
                                    _u16p, C.c_uint16, C.c_int]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_load.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_char_p,
                               C.POINTER(C.c_void_p)]
        L.ref_graph_sizes.argtypes = [C.c_void_p, _u32p, _u64p, _u16p, _u16p, C.POINTER(C.c_int)]
        L.ref_graph_copy.argtypes = [C.c_void_p, _u64p, _u32p, _dp, _u16p, _u16p]
        L.ref_write_edge_list.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_model_new.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, _u16p, C.c_uint32,
                                    _dp, C.c_uint32, C.POINTER(C.c_void_p)]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_decide.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, _u32p, _u32p, _u32p, _u32p,
                                 _dp, _dp, _dp, _u8p]
        L.ref_slot_count.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_slot_count.restype = C.c_uint64
        L.ref_alias_build.argtypes = [C.c_uint32, _dp, _dp, _u32p]
        L.ref_generate_walks.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32,
                                         _u32p, _u32p, _u64p, _u64p, _dp]
        L.ref_walk_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, C.c_uint64,
                                      C.c_uint64, C.c_uint64, _u64p, _dp]
        L.ref_json_double.argtypes = [C.c_double, C.c_char_p, C.c_size_t]
        L.ref_write_corpus.argtypes = [C.c_char_p, _u32p, _u32p, C.c_uint64, C.c_uint32, _u64p, _dp]
        L.ref_manifest.argtypes = [C.POINTER(C.c_char_p), _dp, _u64p, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]
        L.ref_run_new.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                  C.c_int, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]
        L.ref_run_free.argtypes = [C.c_void_p]
        L.ref_run_slice.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, _u64p, _dp]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def json_double(self, x: float) -> str:
        """nlohmann::json(x).dump() (the stats sidecar's number format)."""
        buf = C.create_string_buffer(64)
        self._check(self.lib.ref_json_double(float(x), buf, 64))
        return buf.value.decode()

    def write_corpus(self, path, rows, lens, stats: dict):
        """The reference's write_corpus (engine.cpp:236-259) on a padded corpus."""
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        lens = np.ascontiguousarray(lens, dtype=np.uint32)
        st = np.array([stats["walks"], stats["early_terminations"], stats["skipped_starts"], stats["steps"]],
                      dtype=np.uint64)
        tm = np.array([stats["steps_per_sec"], stats["init_seconds"], stats["walk_seconds"]], dtype=np.float64)
        self._check(self.lib.ref_write_corpus(path.encode(), _ptr(rows, _u32p), _ptr(lens, _u32p), len(lens),
                                              rows.shape[1] if rows.ndim == 2 else 0, _ptr(st, _u64p),
                                              _ptr(tm, _dp)))

    MANIFEST_STRS = ["input", "model", "metapath", "edge_matrix", "node_types", "edge_types", "sampler", "init",
                     "output"]
    MANIFEST_NUMS = ["p", "q", "T_i", "T_w"]
    MANIFEST_INTS = ["walks_per_node", "walk_length", "burn_in_steps", "hw_sample_size", "threads", "seed",
                     "nodes", "arcs", "checksum"]
    MANIFEST_FLAGS = ["weighted", "symmetrize"]

    def manifest(self, **f) -> bytes:
        """cmd_walk's manifest object (tools/mhwalk.cpp:142-169) dumped by
        nlohmann with indent 2, plus a newline."""
        strs = (C.c_char_p * 9)(*[f.get(k, "").encode() for k in self.MANIFEST_STRS])
        nums = np.array([f.get(k, 0.0) for k in self.MANIFEST_NUMS], dtype=np.float64)
        ints = np.array([f.get(k, 0) for k in self.MANIFEST_INTS], dtype=np.uint64)
        flags = (C.c_int * 2)(*[int(f.get(k, 0)) for k in self.MANIFEST_FLAGS])
        buf = C.create_string_buffer(1 << 16)
        self._check(self.lib.ref_manifest(strs, _ptr(nums, _dp), _ptr(ints, _u64p), flags, buf, 1 << 16))
        return buf.value

    def graph(self, g: HostGraph):
        return _RefGraph(self, self.lib.ref_graph_new(
            g.n, g.m, _ptr(g.offsets, _u64p), _ptr(g.nbr, _u32p), _ptr(g.w, _dp),
            _ptr(g.ntype, _u16p), g.n_ntypes, _ptr(g.etype, _u16p), g.n_etypes, int(g.symmetric)))

    def load(self, path, weighted=False, symmetrize=False, ntypes_path=None, etypes_path=None):
        h = C.c_void_p()
        rc = self.lib.ref_load(path.encode(), int(weighted), int(symmetrize),
                               (ntypes_path or "").encode(), (etypes_path or "").encode(), C.byref(h))
        self._check(rc)
        rg = _RefGraph(self, h.value)
        return rg

    def alias_build(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        prob = np.zeros(len(w))
        alias = np.zeros(len(w), dtype=np.uint32)
        self._check(self.lib.ref_alias_build(len(w), _ptr(w, _dp), _ptr(prob, _dp), _ptr(alias, _u32p)))
        return prob, alias


class _RefGraph:
    def __init__(self, ref: RefLib, handle):
        self.ref, self.h = ref, handle

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass

    def to_host(self) -> HostGraph:
        L = self.ref.lib
        n, m, nt, et, sym = C.c_uint32(), C.c_uint64(), C.c_uint16(), C.c_uint16(), C.c_int()
        L.ref_graph_sizes(self.h, C.byref(n), C.byref(m), C.byref(nt), C.byref(et), C.byref(sym))
        off = np.zeros(n.value + 1, dtype=np.uint64)
        nb = np.zeros(m.value, dtype=np.uint32)
        w = np.zeros(m.value)
        ntype = np.zeros(n.value, dtype=np.uint16) if nt.value else None
        etype = np.zeros(m.value, dtype=np.uint16) if et.value else None
        L.ref_graph_copy(self.h, _ptr(off, _u64p), _ptr(nb, _u32p), _ptr(w, _dp), _ptr(ntype, _u16p),
                         _ptr(etype, _u16p))
        return HostGraph(off, nb, w, ntype, etype, nt.value, et.value, bool(sym.value))

    def write_edge_list(self, path):
        self.ref._check(self.ref.lib.ref_write_edge_list(self.h, path.encode()))

    def model(self, md: ModelDesc):
        h = C.c_void_p()
        mp = np.ascontiguousarray(md.metapath, dtype=np.uint16) if md.metapath else None
        M = None if md.type_matrix is None else np.ascontiguousarray(md.type_matrix, dtype=np.float64)
        rc = self.ref.lib.ref_model_new(self.h, md.kind, md.p, md.q, _ptr(mp, _u16p),
                                        0 if mp is None else len(mp), _ptr(M, _dp),
                                        0 if M is None else M.shape[0], C.byref(h))
        self.ref._check(rc)
        return _RefModel(self, h.value)


class _RefModel:
    def __init__(self, g: _RefGraph, handle):
        self.g, self.h = g, handle

    def __del__(self):
        try:
            self.g.ref.lib.ref_model_free(self.h)
        except Exception:
            pass

    def decide(self, pos, affix, cand, last, u):
        n = len(pos)
        arrs = [np.ascontiguousarray(x, dtype=np.uint32) for x in (pos, affix, cand, last)]
        uu = np.ascontiguousarray(u, dtype=np.float64)
        wc, wl = np.zeros(n), np.zeros(n)
        acc = np.zeros(n, dtype=np.uint8)
        self.g.ref.lib.ref_decide(self.g.h, self.h, n, *[_ptr(a, _u32p) for a in arrs],
                                  _ptr(uu, _dp), _ptr(wc, _dp), _ptr(wl, _dp), _ptr(acc, _u8p))
        return wc, wl, acc

    def slot_count(self):
        return self.g.ref.lib.ref_slot_count(self.g.h, self.h)

    def generate_walks(self, cfg: WalkCfg, threads=1, n_nodes=None, with_rows=True):
        L = self.g.ref.lib
        n = n_nodes if n_nodes is not None else self.g.to_host().n
        stride = cfg.L + 1
        total = max(n * cfg.K, 1)
        rows = np.zeros((total, stride), dtype=np.uint32) if with_rows else None
        lens = np.zeros(total, dtype=np.uint32) if with_rows else None
        nrows = C.c_uint64()
        st = np.zeros(4, dtype=np.uint64)
        tm = np.zeros(3)
        rc = L.ref_generate_walks(self.g.h, self.h, cfg.K, cfg.L, threads, cfg.seed, cfg.init_kind,
                                  cfg.burn_in_steps, cfg.hw_sample_size, cfg.sampler, stride, _ptr(rows, _u32p),
                                  _ptr(lens, _u32p), C.byref(nrows), _ptr(st, _u64p), _ptr(tm, _dp))
        self.g.ref._check(rc)
        stats = dict(walks=int(st[0]), early_terminations=int(st[1]), skipped_starts=int(st[2]),
                     steps=int(st[3]), seconds=float(tm[0]), init_seconds=float(tm[1]),
                     steps_per_sec=float(tm[2]))
        k = nrows.value
        if with_rows:
            return rows[:k], lens[:k], stats
        return None, None, stats

    def walk_sample(self, cfg: WalkCfg, begin, stride, count, threads):
        st = np.zeros(4, dtype=np.uint64)
        tm = np.zeros(2)
        rc = self.g.ref.lib.ref_walk_sample(self.g.h, self.h, cfg.K, cfg.L, threads, cfg.seed,
                                            cfg.init_kind, cfg.burn_in_steps, cfg.hw_sample_size,
                                            begin, stride, count, _ptr(st, _u64p), _ptr(tm, _dp))
        self.g.ref._check(rc)
        return dict(walks=int(st[0]), early_terminations=int(st[1]), skipped_starts=int(st[2]),
                    steps=int(st[3]), seconds=float(tm[0]), init_seconds=float(tm[1]))

    def full_run(self, cfg: WalkCfg, threads):
        """One generate_walks-equivalent run over ALL walkers with one shared
        SamplerManager, executed in time slices (ref_run_slice)."""
        return _RefRun(self, cfg, threads)


class _RefRun:
    def __init__(self, m: _RefModel, cfg: WalkCfg, threads):
        self.m = m
        L = m.g.ref.lib
        h = C.c_void_p()
        m.g.ref._check(L.ref_run_new(m.g.h, m.h, cfg.K, cfg.L, threads, cfg.seed, cfg.init_kind,
                                     cfg.burn_in_steps, cfg.hw_sample_size, C.byref(h)))
        self.h = h.value

    def slice(self, i, n):
        st = np.zeros(4, dtype=np.uint64)
        tm = np.zeros(2)
        self.m.g.ref._check(self.m.g.ref.lib.ref_run_slice(self.h, i, n, _ptr(st, _u64p), _ptr(tm, _dp)))
        return dict(walks=int(st[0]), early_terminations=int(st[1]), skipped_starts=int(st[2]),
                    steps=int(st[3]), seconds=float(tm[0]), init_seconds=float(tm[1]))

    def __del__(self):
        try:
            self.m.g.ref.lib.ref_run_free(self.h)
        except Exception:
            pass


# ------------------------------------------------------------ test graphs
def xo_rng(seed):
    """Tiny Python xoshiro256** for restating the reference's test builders
    (tests/oracles.hpp:27-118) without calling the library."""
    return XoRng(seed)


class XoRng:
    M64 = (1 << 64) - 1

    def __init__(self, seed):
        sm = [seed & self.M64]
        self.s = [self._sm(sm) for _ in range(4)]

    def _sm(self, st):
        st[0] = (st[0] + 0x9E3779B97F4A7C15) & self.M64
        z = st[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M64
        return z ^ (z >> 31)

    def next(self):
        s = self.s
        rot = lambda x, k: ((x << k) | (x >> (64 - k))) & self.M64
        result = (rot((s[1] * 5) & self.M64, 7) * 9) & self.M64
        t = (s[1] << 17) & self.M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = rot(s[3], 45)
        return result

    def uniform_index(self, n):
        x = self.next() >> 32
        m = x * n
        lo = m & 0xFFFFFFFF
        if lo < n:
            thr = ((1 << 32) - n) % n
            while lo < thr:
                x = self.next() >> 32
                m = x * n
                lo = m & 0xFFFFFFFF
        return m >> 32

    def uniform_real(self):
        return (self.next() >> 11) * 2.0 ** -53


def make_graph(n, edges, symmetric=True) -> HostGraph:
    """oracles::make_graph (tests/oracles.hpp:27-40)."""
    edges = sorted(edges)
    off = np.zeros(n + 1, dtype=np.uint64)
    for u, _, _ in edges:
        off[u + 1] += 1
    off = np.cumsum(off, dtype=np.uint64)
    nb = np.array([v for _, v, _ in edges], dtype=np.uint32)
    w = np.array([x for _, _, x in edges], dtype=np.float64)
    return HostGraph(off, nb, w, symmetric=symmetric)


def triangle() -> HostGraph:
    return make_graph(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 0, 1.0), (1, 2, 1.0), (2, 0, 1.0), (2, 1, 1.0)])


def random_graph(n, avg_deg, weighted, rng: XoRng, ensure_connected=True, f32=True) -> HostGraph:
    """oracles::random_graph (tests/oracles.hpp:50-68). Weights are rounded to
    fp32 when f32=True so the device CSR (fp32 weights) holds the same values."""
    seen = set()
    edges = []

    def add(a, b):
        if a == b:
            return
        if a > b:
            a, b = b, a
        if (a, b) in seen:
            return
        seen.add((a, b))
        w = 0.1 + 1.9 * rng.uniform_real() if weighted else 1.0
        if f32:
            w = float(np.float32(w))
        edges.append((a, b, w))
        edges.append((b, a, w))

    if ensure_connected:
        for v in range(1, n):
            add(v, rng.uniform_index(v))
    extra = int(n * avg_deg / 2)
    for _ in range(extra):
        add(rng.uniform_index(n), rng.uniform_index(n))
    return make_graph(n, edges)


def preferential_attachment(n, m, rng: XoRng) -> HostGraph:
    """oracles::preferential_attachment (tests/oracles.hpp:72-94)."""
    endpoints, seen, edges = [], set(), []

    def add(a, b):
        if a == b:
            return False
        key = (min(a, b), max(a, b))
        if key in seen:
            return False
        seen.add(key)
        edges.append((a, b, 1.0))
        edges.append((b, a, 1.0))
        endpoints.extend([a, b])
        return True

    v = 1
    while v <= m and v < n:
        add(v, 0)
        v += 1
    for v in range(m + 1, n):
        for _ in range(m):
            add(v, endpoints[rng.uniform_index(len(endpoints))])
    return make_graph(n, edges)


def star(leaves) -> HostGraph:
    """oracles::star (tests/oracles.hpp:97-104)."""
    edges = []
    for v in range(1, leaves + 1):
        edges += [(0, v, 1.0), (v, 0, 1.0)]
    return make_graph(leaves + 1, edges)


def assign_random_types(g: HostGraph, num_types, rng: XoRng):
    """oracles::assign_random_types (tests/oracles.hpp:106-112)."""
    t = np.array([rng.uniform_index(num_types) for _ in range(g.n)], dtype=np.uint16)
    for i in range(min(num_types, g.n)):
        t[i] = i
    g.ntype = t
    g.n_ntypes = num_types


def eval_target(g: HostGraph, oracle: Oracle, md: ModelDesc, v, affix):
    """Exact normalised w' at state (v, affix) (tools/mhwalk.cpp:208-220)."""
    d = g.degree(v)
    idx = np.arange(d, dtype=np.uint32)
    wc, _, _ = oracle.decide(g, md, np.full(d, v), np.full(d, affix), idx, idx, np.zeros(d))
    t = wc.sum()
    return wc / t if t > 0 else wc
