"""Python mirror of the reference's walk-path API (namespace mhwalk of
/root/reference/proj) over the C ABI of libmhw.so.

Same names, argument meanings and error classes as the reference:
  Graph            graph.hpp:15-55      (device-resident CSR handle)
  load_edge_list   graph.hpp:65 / graph.cpp:70-100
  ModelKind        models.hpp:13         WalkModel  models.hpp:40-92
  InitStrategy     samplers.hpp:29-34    SamplerKind engine.hpp:12
  WalkConfig       engine.hpp:19-26      RunStats   engine.hpp:28-36
  WalkCorpus       engine.hpp:38-41      generate_walks engine.hpp:47
  write_corpus / read_corpus  engine.hpp:50-52
  ParseError / ValidationError / IoError  errors.hpp:8-21
WalkConfig.threads == 1 selects the deterministic schedule (the GPU
counterpart of the reference's single-thread byte determinism,
engine.hpp:43-46); any other value selects the throughput schedule.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class MhwError(RuntimeError):
    code = 4


class IoError(MhwError):
    code = 1


class ValidationError(MhwError):
    code = 2


class ParseError(ValidationError):
    code = 2


class CudaError(MhwError):
    code = 4


def _check(rc: int):
    if rc == 0:
        return
    msg = L.lib().mhw_last_error().decode()
    if rc == 1:
        raise IoError(msg)
    if rc == 2:
        raise ValidationError(msg)
    raise CudaError(msg)


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class ModelKind(enum.IntEnum):
    deepwalk = 0
    node2vec = 1
    metapath2vec = 2
    edge2vec = 3
    fairwalk = 4


def model_kind_from_string(name: str) -> ModelKind:
    try:
        return ModelKind[name]
    except KeyError:
        raise ValidationError(f"unknown model: {name}") from None


class InitKind(enum.IntEnum):
    random = 0
    high_weight = 1
    burn_in = 2


def init_kind_from_string(name: str) -> InitKind:
    key = name.replace("-", "_")
    try:
        return InitKind[key]
    except KeyError:
        raise ValidationError(f"unknown init strategy: {name}") from None


class SamplerKind(enum.IntEnum):
    mh = 0
    alias = 1
    direct = 2
    rejection = 3


class Schedule(enum.IntEnum):
    throughput = 0
    deterministic = 1


kNoAffix = 0xFFFFFFFF


@dataclass
class InitStrategy:
    kind: InitKind = InitKind.random
    burn_in_steps: int = 100
    hw_sample_size: int = 32


@dataclass
class WalkModel:
    kind: ModelKind = ModelKind.deepwalk
    p: float = 1.0
    q: float = 1.0
    metapath: list = field(default_factory=list)
    type_matrix: list | np.ndarray | None = None

    def second_order(self) -> bool:
        return self.kind in (ModelKind.node2vec, ModelKind.edge2vec, ModelKind.fairwalk)

    def _desc(self):
        d = L.ModelDescC()
        keep = []
        d.kind, d.p, d.q = int(self.kind), float(self.p), float(self.q)
        if self.metapath:
            mp = np.ascontiguousarray(self.metapath, dtype=np.uint16)
            keep.append(mp)
            d.metapath, d.metapath_len = mp.ctypes.data, len(mp)
        if self.type_matrix is not None:
            M = np.ascontiguousarray(self.type_matrix, dtype=np.float64)
            if M.ndim != 2 or M.shape[0] != M.shape[1]:
                raise ValidationError("edge type matrix is not square")
            keep.append(M)
            d.type_matrix, d.type_matrix_dim = M.ctypes.data, M.shape[0]
        return d, keep


@dataclass
class WalkConfig:
    walks_per_node: int = 10
    walk_length: int = 80
    threads: int = 1
    seed: int = 0
    sampler_kind: SamplerKind = SamplerKind.mh
    init: InitStrategy = field(default_factory=InitStrategy)
    schedule: Schedule | None = None   # None: derived from threads
    node_begin: int = 0
    node_end: int = 0
    chain_replica_degree: int = 0      # 0: auto; 0xFFFFFFFF: one chain per state
    init_mode: int = 0                 # 0 auto, 1 lazy, 2 eager
    proposal: int = 0                  # 0 uniform (samplers.hpp:21), 1 static-weight alias + Hastings

    def _c(self):
        c = L.WalkConfigC()
        if self.threads == 0:
            raise ValidationError("walks_per_node, walk_length and threads must be positive")
        c.walks_per_node, c.walk_length, c.seed = self.walks_per_node, self.walk_length, self.seed
        c.sampler = int(self.sampler_kind)
        c.init_kind = int(self.init.kind)
        c.burn_in_steps, c.hw_sample_size = self.init.burn_in_steps, self.init.hw_sample_size
        sched = self.schedule
        if sched is None:
            sched = Schedule.deterministic if self.threads == 1 else Schedule.throughput
        c.schedule = int(sched)
        c.node_begin, c.node_end = self.node_begin, self.node_end
        c.chain_replica_degree, c.init_mode = self.chain_replica_degree, self.init_mode
        c.proposal = int(self.proposal)
        return c


@dataclass
class RunStats:
    walks: int = 0
    early_terminations: int = 0
    skipped_starts: int = 0
    steps: int = 0
    steps_per_sec: float = 0.0
    init_seconds: float = 0.0
    walk_seconds: float = 0.0
    slot_inits: int = 0
    chain_retries: int = 0
    rejection_trials: int = 0

    @classmethod
    def _from(cls, s: L.WalkStatsC):
        return cls(s.walks, s.early_terminations, s.skipped_starts, s.steps, s.steps_per_sec, s.init_seconds,
                   s.walk_seconds, s.slot_inits, s.chain_retries, s.rejection_trials)


class WalkCorpus:
    """Padded corpus: rows[r, :lengths[r]] is walk r (reference corpus order)."""

    def __init__(self, rows: np.ndarray, lengths: np.ndarray, stats: RunStats):
        self.rows, self.lengths, self.stats = rows, lengths, stats

    @property
    def walks(self):
        return [self.rows[r, :self.lengths[r]] for r in range(len(self.lengths))]

    def __len__(self):
        return len(self.lengths)


class Graph:
    """Device-resident CSR (one replica on one device)."""

    def __init__(self, handle, device=0):
        self._h = C.c_void_p(handle)
        self.device = device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().mhw_graph_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    # ------------------------------------------------------------ builders
    @classmethod
    def from_csr(cls, offsets, neighbors, weights=None, node_types=None, edge_types=None, symmetric=True,
                 num_node_types=0, num_edge_types=0, device=0) -> "Graph":
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        nb = np.ascontiguousarray(neighbors, dtype=np.int32)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float32)
        nt = None if node_types is None else np.ascontiguousarray(node_types, dtype=np.uint16)
        et = None if edge_types is None else np.ascontiguousarray(edge_types, dtype=np.uint16)
        v = L.GraphView()
        v.node_count, v.arc_count = len(off) - 1, len(nb)
        v.offsets, v.neighbors = off.ctypes.data, (nb.ctypes.data if len(nb) else None)
        v.weights = None if w is None else w.ctypes.data
        v.node_types = None if nt is None else nt.ctypes.data
        v.edge_types = None if et is None else et.ctypes.data
        v.num_node_types, v.num_edge_types, v.symmetric = num_node_types, num_edge_types, int(symmetric)
        h = C.c_void_p()
        _check(L.lib().mhw_graph_upload(C.byref(v), device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def from_host(cls, hg, device=0, weighted=True) -> "Graph":
        """From an oracle.HostGraph-like object (offsets/nbr/w/ntype/etype)."""
        return cls.from_csr(hg.offsets.astype(np.int64), hg.nbr.astype(np.int32),
                            hg.w.astype(np.float32) if weighted else None, hg.ntype, hg.etype, hg.symmetric,
                            hg.n_ntypes, hg.n_etypes, device)

    @classmethod
    def from_edges(cls, src, dst, weights=None, symmetrize=False, node_count=0, device=0) -> "Graph":
        s = np.ascontiguousarray(src, dtype=np.uint32)
        d = np.ascontiguousarray(dst, dtype=np.uint32)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float32)
        h = C.c_void_p()
        _check(L.lib().mhw_graph_from_edges(len(s), _ptr(s), _ptr(d), _ptr(w), int(symmetrize), node_count,
                                            device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def rmat(cls, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, weighted=False, weight_lo=1.0,
             weight_hi=10.0, edge_types=0, device=0) -> "Graph":
        h = C.c_void_p()
        _check(L.lib().mhw_graph_generate_rmat(scale, edge_factor, a, b, c, seed, int(weighted), weight_lo,
                                               weight_hi, edge_types, device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def hetero(cls, node_count, seed=1, weight_lo=1.0, weight_hi=5.0, device=0) -> "Graph":
        h = C.c_void_p()
        _check(L.lib().mhw_graph_generate_hetero(node_count, seed, weight_lo, weight_hi, device, C.byref(h)))
        return cls(h.value, device)

    # ------------------------------------------------------------- queries
    def info(self) -> dict:
        i = L.GraphInfoC()
        _check(L.lib().mhw_graph_info_get(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in L.GraphInfoC._fields_}

    def checksum(self) -> int:
        """graph_checksum (tools/mhwalk.cpp:107-122) of this CSR."""
        c = C.c_uint64()
        _check(L.lib().mhw_graph_checksum(self._h, C.byref(c)))
        return c.value

    def node_count(self) -> int:
        return self.info()["node_count"]

    def arc_count(self) -> int:
        return self.info()["arc_count"]

    def download(self) -> dict:
        inf = self.info()
        n, m = inf["node_count"], inf["arc_count"]
        off = np.zeros(n + 1, dtype=np.int64)
        nb = np.zeros(max(m, 1), dtype=np.int32)
        w = np.zeros(max(m, 1), dtype=np.float32)
        nt = np.zeros(max(n, 1), dtype=np.uint16) if inf["num_node_types"] else None
        et = np.zeros(max(m, 1), dtype=np.uint16) if inf["num_edge_types"] else None
        _check(L.lib().mhw_graph_download(self._h, _ptr(off), _ptr(nb), _ptr(w), _ptr(nt), _ptr(et)))
        return dict(offsets=off, neighbors=nb[:m], weights=w[:m] if inf["weighted"] else None,
                    node_types=None if nt is None else nt[:n], edge_types=None if et is None else et[:m],
                    num_node_types=inf["num_node_types"], num_edge_types=inf["num_edge_types"])

    def set_node_types(self, types, num_types=0):
        t = np.ascontiguousarray(types, dtype=np.uint16)
        _check(L.lib().mhw_graph_set_node_types(self._h, _ptr(t), num_types))

    def set_edge_types(self, types, num_types=0):
        t = np.ascontiguousarray(types, dtype=np.uint16)
        _check(L.lib().mhw_graph_set_edge_types(self._h, _ptr(t), num_types))

    def replicate(self, device) -> "Graph":
        h = C.c_void_p()
        _check(L.lib().mhw_graph_replicate(self._h, device, C.byref(h)))
        return Graph(h.value, device)


def load_edge_list(path, weighted=False, symmetrize=False, device=0) -> Graph:
    """load_edge_list (graph.cpp:70-100) through the native multi-threaded
    parser + device build_csr: "src dst [weight]" lines, '#' comments;
    ParseError / ValidationError with "path:LINE: ..." messages, IoError for
    an unreadable file."""
    h = C.c_void_p()
    rc = L.lib().mhw_graph_load_edge_list(str(path).encode(), int(weighted), int(symmetrize), device, C.byref(h))
    if rc == 2:
        msg = L.lib().mhw_last_error().decode()
        if "negative" in msg:
            raise ValidationError(msg)
        raise ParseError(msg)
    _check(rc)
    return Graph(h.value, device)


def load_node_types(graph: Graph, path):
    """load_node_types (graph.cpp:102-135)."""
    _check(L.lib().mhw_graph_load_node_types(graph.handle, str(path).encode()))


def load_edge_types(graph: Graph, path):
    """load_edge_types (graph.cpp:137-177); symmetric graphs type both directions."""
    _check(L.lib().mhw_graph_load_edge_types(graph.handle, str(path).encode()))


def generate_walks(graph: Graph, model: WalkModel, config: WalkConfig) -> WalkCorpus:
    """generate_walks (engine.cpp:157-234) on the GPU."""
    d, keep = model._desc()
    c = config._c()
    h = C.c_void_p()
    _check(L.lib().mhw_generate_walks(graph.handle, C.byref(d), C.byref(c), C.byref(h)))
    lib = L.lib()
    try:
        rows, stride = lib.mhw_walks_count(h), lib.mhw_walks_stride(h)
        st = L.WalkStatsC()
        _check(lib.mhw_walks_stats(h, C.byref(st)))
        nodes = np.zeros((rows, stride), dtype=np.uint32)
        lens = np.zeros(rows, dtype=np.uint32)
        if rows:
            C.memmove(nodes.ctypes.data, lib.mhw_walks_nodes(h), rows * stride * 4)
            C.memmove(lens.ctypes.data, lib.mhw_walks_lengths(h), rows * 4)
    finally:
        lib.mhw_walks_free(h)
    return WalkCorpus(nodes, lens, RunStats._from(st))


def generate_walks_packed(graph: Graph, model: WalkModel, config: WalkConfig):
    """generate_walks into a packed corpus: (nodes, offsets, RunStats) with
    walk r = nodes[offsets[r]:offsets[r+1]] (compacted on the device)."""
    d, keep = model._desc()
    c = config._c()
    lib = L.lib()
    rows, stride = C.c_uint64(), C.c_uint32()
    _check(lib.mhw_walk_rows(graph.handle, C.byref(d), C.byref(c), C.byref(rows), C.byref(stride)))
    cap = max(rows.value * (config.walk_length + 1), 1)
    nodes = np.zeros(cap, dtype=np.uint32)
    offsets = np.zeros(rows.value + 1, dtype=np.uint64)
    st = L.WalkStatsC()
    _check(lib.mhw_generate_walks_packed(graph.handle, C.byref(d), C.byref(c), _ptr(nodes), cap, _ptr(offsets),
                                         rows.value + 1, C.byref(st)))
    return nodes[:int(offsets[-1])], offsets, RunStats._from(st)


def generate_walks_multi(replicas: list, model: WalkModel, config: WalkConfig) -> WalkCorpus:
    d, keep = model._desc()
    c = config._c()
    arr = (C.c_void_p * len(replicas))(*[g.handle.value for g in replicas])
    h = C.c_void_p()
    _check(L.lib().mhw_generate_walks_multi(C.cast(arr, C.c_void_p), len(replicas), C.byref(d), C.byref(c),
                                            C.byref(h)))
    lib = L.lib()
    try:
        rows, stride = lib.mhw_walks_count(h), lib.mhw_walks_stride(h)
        st = L.WalkStatsC()
        _check(lib.mhw_walks_stats(h, C.byref(st)))
        nodes = np.zeros((rows, stride), dtype=np.uint32)
        lens = np.zeros(rows, dtype=np.uint32)
        if rows:
            C.memmove(nodes.ctypes.data, lib.mhw_walks_nodes(h), rows * stride * 4)
            C.memmove(lens.ctypes.data, lib.mhw_walks_lengths(h), rows * 4)
    finally:
        lib.mhw_walks_free(h)
    return WalkCorpus(nodes, lens, RunStats._from(st))


def partition_nodes(graph: Graph, model: WalkModel, parts: int) -> np.ndarray:
    d, keep = model._desc()
    cuts = np.zeros(parts + 1, dtype=np.uint32)
    _check(L.lib().mhw_partition_nodes(graph.handle, C.byref(d), parts, _ptr(cuts)))
    return cuts


def write_corpus(corpus: WalkCorpus, path: str):
    """write_corpus (engine.cpp:236-259): one walk per line + stats sidecar."""
    try:
        with open(path, "w") as f:
            for r in range(len(corpus.lengths)):
                f.write(" ".join(map(str, corpus.rows[r, :corpus.lengths[r]].tolist())))
                f.write("\n")
    except OSError:
        raise IoError(f"cannot open for writing: {path}") from None
    with open(path + ".stats.jsonl", "wb") as f:
        f.write(stats_line(corpus.stats))


def _stats_c(s) -> "L.WalkStatsC":
    c = L.WalkStatsC()
    for k, _ in L.WalkStatsC._fields_:
        setattr(c, k, getattr(s, k, 0))
    return c


def stats_line(stats) -> bytes:
    """The `.stats.jsonl` line of write_corpus (engine.cpp:248-259) as the
    reference's nlohmann dump() renders it (mhw_stats_render)."""
    c = _stats_c(stats)
    n = C.c_size_t()
    _check(L.lib().mhw_stats_render(C.byref(c), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(L.lib().mhw_stats_render(C.byref(c), buf, n.value + 1, C.byref(n)))
    return buf.raw[:n.value]


MANIFEST_FIELDS = [k for k, _ in L.ManifestC._fields_]


def _manifest_c(fields: dict):
    m = L.ManifestC()
    for k, t in L.ManifestC._fields_:
        v = fields.get(k, "" if t is C.c_char_p else 0)
        setattr(m, k, v.encode() if t is C.c_char_p else v)
    return m


def render_manifest(**fields) -> bytes:
    """cmd_walk's `.manifest.json` (tools/mhwalk.cpp:142-169), nlohmann
    dump(2) layout (mhw_manifest_render). Fields: mhw_manifest's."""
    m = _manifest_c(fields)
    n = C.c_size_t()
    _check(L.lib().mhw_manifest_render(C.byref(m), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(L.lib().mhw_manifest_render(C.byref(m), buf, n.value + 1, C.byref(n)))
    return buf.raw[:n.value]


def write_manifest(graph: "Graph", model: "WalkModel", config: "WalkConfig", stats, output: str, input: str = "",
                   weighted: bool = False, symmetrize: bool = False, metapath: str = "", edge_matrix: str = "",
                   node_types: str = "", edge_types: str = ""):
    """The run manifest cmd_walk writes beside the corpus
    (<output>.manifest.json: config flags, graph size + checksum, T_i/T_w)."""
    info = graph.info()
    fields = dict(input=input, weighted=int(weighted), symmetrize=int(symmetrize), model=model.kind.name,
                  p=model.p, q=model.q, metapath=metapath, edge_matrix=edge_matrix, node_types=node_types,
                  edge_types=edge_types, walks_per_node=config.walks_per_node, walk_length=config.walk_length,
                  sampler=config.sampler_kind.name, init=config.init.kind.name,
                  burn_in_steps=config.init.burn_in_steps, hw_sample_size=config.init.hw_sample_size,
                  threads=config.threads, seed=config.seed, output=output, nodes=info["node_count"],
                  arcs=info["arc_count"], checksum=graph.checksum(), T_i=stats.init_seconds,
                  T_w=stats.walk_seconds)
    m = _manifest_c(fields)
    _check(L.lib().mhw_manifest_write(C.byref(m)))


def read_corpus(path: str) -> list:
    """read_corpus (engine.cpp:261-275)."""
    if not os.path.exists(path):
        raise IoError(f"cannot open corpus: {path}")
    out = []
    with open(path) as f:
        for line in f:
            w = [int(x) for x in line.split()]
            if w:
                out.append(w)
    return out


# --------------------------------------------------------- parity helpers
def decide(graph: Graph, model: WalkModel, position, affixture, candidate, last, u):
    """(state, cand, last, u) -> (w'(cand), w'(last), accept) on the GPU."""
    d, keep = model._desc()
    arrs = [np.ascontiguousarray(x, dtype=np.uint32) for x in (position, affixture, candidate, last)]
    uu = np.ascontiguousarray(u, dtype=np.float64)
    n = len(uu)
    wc, wl = np.zeros(max(n, 1)), np.zeros(max(n, 1))
    acc = np.zeros(max(n, 1), dtype=np.uint8)
    _check(L.lib().mhw_decide(graph.handle, C.byref(d), n, *[_ptr(a) for a in arrs], _ptr(uu), _ptr(wc),
                              _ptr(wl), _ptr(acc)))
    return wc[:n], wl[:n], acc[:n]


def decide_hastings(graph: Graph, model: WalkModel, position, affixture, candidate, last, u):
    """Alias-proposal decisions on the GPU: (r(cand), r(last), accept) with
    r = w'/w and the Hastings accept (mhw_decide_hastings)."""
    d, keep = model._desc()
    arrs = [np.ascontiguousarray(x, dtype=np.uint32) for x in (position, affixture, candidate, last)]
    uu = np.ascontiguousarray(u, dtype=np.float64)
    n = len(uu)
    rc, rl = np.zeros(max(n, 1)), np.zeros(max(n, 1))
    acc = np.zeros(max(n, 1), dtype=np.uint8)
    _check(L.lib().mhw_decide_hastings(graph.handle, C.byref(d), n, *[_ptr(a) for a in arrs], _ptr(uu), _ptr(rc),
                                       _ptr(rl), _ptr(acc)))
    return rc[:n], rl[:n], acc[:n]


def check(graph: Graph, model: WalkModel, position, affixture, draws: int, seed: int = 0,
          tolerance: float | None = None):
    """cmd_check (tools/mhwalk.cpp:222-264) on the GPU: per-state KL of a
    `draws`-long M-H chain against the exact target. Returns (kl, counts,
    exit_code) with exit_code = 0 if max KL < tolerance else 3 (None without
    a tolerance)."""
    d, keep = model._desc()
    pos = np.ascontiguousarray(position, dtype=np.uint32)
    aff = np.ascontiguousarray(affixture, dtype=np.uint32)
    n = len(pos)
    kl = np.zeros(max(n, 1))
    total = 0
    if n:
        offs = graph.download()["offsets"]
        total = int(np.sum(offs[pos.astype(np.int64) + 1] - offs[pos.astype(np.int64)]))
    counts = np.zeros(max(total, 1), dtype=np.uint64)
    _check(L.lib().mhw_check(graph.handle, C.byref(d), seed, n, _ptr(pos), _ptr(aff), draws, _ptr(kl),
                             _ptr(counts)))
    kl = kl[:n]
    code = None
    if tolerance is not None:
        valid = kl[~np.isnan(kl)]
        code = 0 if (valid.max() if len(valid) else 0.0) < tolerance else 3
    return kl, counts[:total], code


def alias_tables(graph: Graph):
    m = graph.arc_count()
    prob = np.zeros(max(m, 1))
    alias = np.zeros(max(m, 1), dtype=np.uint32)
    _check(L.lib().mhw_alias_tables(graph.handle, _ptr(prob), _ptr(alias)))
    return prob[:m], alias[:m]


def init_states(graph: Graph, model: WalkModel, config: WalkConfig, position, affixture):
    d, keep = model._desc()
    c = config._c()
    pos = np.ascontiguousarray(position, dtype=np.uint32)
    aff = np.ascontiguousarray(affixture, dtype=np.uint32)
    out = np.zeros(max(len(pos), 1), dtype=np.uint32)
    _check(L.lib().mhw_init_states(graph.handle, C.byref(d), C.byref(c), len(pos), _ptr(pos), _ptr(aff),
                                   _ptr(out)))
    return out[:len(pos)]


class Session:
    """Device-resident repeated generate_walks (benchmarks)."""

    def __init__(self, graph: Graph, model: WalkModel, config: WalkConfig):
        self._d, self._keep = model._desc()
        self._c = config._c()
        self.graph = graph
        h = C.c_void_p()
        _check(L.lib().mhw_session_create(graph.handle, C.byref(self._d), C.byref(self._c), C.byref(h)))
        self._h = h
        rows, stride = C.c_uint64(), C.c_uint32()
        dn, dl = C.c_void_p(), C.c_void_p()
        _check(L.lib().mhw_session_buffers(h, C.byref(dn), C.byref(dl), C.byref(rows), C.byref(stride)))
        self.rows, self.stride = rows.value, stride.value
        self.d_nodes, self.d_lengths = dn.value, dl.value

    def run(self, stream: int | None = None):
        _check(L.lib().mhw_session_run(self._h, C.c_void_p(stream) if stream else None))

    def select_starts(self, starts=None):
        """Restrict the next runs to these (ascending) start nodes; None = the
        whole node range (mhw_session_select_starts)."""
        if starts is None:
            _check(L.lib().mhw_session_select_starts(self._h, 0, None))
        else:
            a = np.ascontiguousarray(starts, dtype=np.uint32)
            _check(L.lib().mhw_session_select_starts(self._h, len(a), _ptr(a) if len(a) else None))
        rows, stride = C.c_uint64(), C.c_uint32()
        dn, dl = C.c_void_p(), C.c_void_p()
        _check(L.lib().mhw_session_buffers(self._h, C.byref(dn), C.byref(dl), C.byref(rows), C.byref(stride)))
        self.rows = rows.value

    def stats(self) -> RunStats:
        st = L.WalkStatsC()
        _check(L.lib().mhw_session_stats(self._h, C.byref(st)))
        return RunStats._from(st)

    def launches(self) -> int:
        return L.lib().mhw_session_launches(self._h)

    # sharded chain initialisation (multi-GPU): see include/mhw.h
    def chain_size(self) -> int:
        n = C.c_uint64()
        _check(L.lib().mhw_session_chain_size(self._h, C.byref(n)))
        return n.value

    def init_chain(self, begin: int, end: int, d_words: int, stream: int | None = None):
        """Initial words of slots [begin, end) into device memory d_words."""
        _check(L.lib().mhw_session_init_chain(self._h, begin, end, C.c_void_p(d_words),
                                              C.c_void_p(stream) if stream else None))

    def load_chain(self, d_words: int, stream: int | None = None):
        """Installs a full initial table (chain_size words) for the next run."""
        _check(L.lib().mhw_session_load_chain(self._h, C.c_void_p(d_words), C.c_void_p(stream) if stream else None))

    def shard_entry_bytes(self) -> int:
        """Bytes per entry of the session's shard exchange (2: compact chains, slot order)."""
        b = C.c_uint32()
        _check(L.lib().mhw_session_shard_entry_bytes(self._h, C.byref(b)))
        return b.value

    def init_shard(self, begin: int, end: int, d_out: int, stream: int | None = None):
        """Entries [begin, end) of the sharded-init exchange (mhw_session_init_shard)."""
        _check(L.lib().mhw_session_init_shard(self._h, begin, end, C.c_void_p(d_out),
                                              C.c_void_p(stream) if stream else None))

    def load_shard_range(self, begin: int, end: int, d_in: int, stream: int | None = None):
        """Installs exchange entries [begin, end) (d_in -> entry begin) for the next run."""
        _check(L.lib().mhw_session_load_shard_range(self._h, begin, end, C.c_void_p(d_in),
                                                    C.c_void_p(stream) if stream else None))

    def prepare(self, stream: int | None = None):
        """Reset + eager init of the session's own table without a walk; the
        next run starts from it (mhw_session_prepare)."""
        _check(L.lib().mhw_session_prepare(self._h, C.c_void_p(stream) if stream else None))

    def export_table(self, d_words: int, stream: int | None = None):
        """The installed chain table, one u32 per arc (chain_size entries)."""
        _check(L.lib().mhw_session_export_table(self._h, C.c_void_p(d_words), C.c_void_p(stream) if stream else None))

    def init_records(self, begin: int, end: int, d_words: int, stream: int | None = None):
        """Initial words of records (arcs) [begin, end): the chain table in the
        order the session stores it (coalesced install by load_records)."""
        _check(L.lib().mhw_session_init_records(self._h, begin, end, C.c_void_p(d_words),
                                                C.c_void_p(stream) if stream else None))

    def record_width(self) -> int:
        """u32 words per entry of a record-order table (3 for typed records)."""
        w = C.c_uint32()
        _check(L.lib().mhw_session_record_width(self._h, C.byref(w)))
        return w.value

    def load_records_range(self, begin: int, end: int, d_words: int, stream: int | None = None):
        """Installs entries [begin, end) of a record-order table (d_words -> entry begin)."""
        _check(L.lib().mhw_session_load_records_range(self._h, begin, end, C.c_void_p(d_words),
                                                      C.c_void_p(stream) if stream else None))

    def load_records(self, d_words: int, stream: int | None = None):
        """Installs a full record-order table for the next run."""
        _check(L.lib().mhw_session_load_records(self._h, C.c_void_p(d_words), C.c_void_p(stream) if stream else None))

    def download(self, nodes=None, lengths=None, stream: int | None = None):
        if nodes is None:
            nodes = np.zeros((self.rows, self.stride), dtype=np.uint32)
        if lengths is None:
            lengths = np.zeros(self.rows, dtype=np.uint32)
        _check(L.lib().mhw_session_download(self._h, C.c_void_p(nodes.ctypes.data) if self.rows else None,
                                            C.c_void_p(lengths.ctypes.data) if self.rows else None,
                                            C.c_void_p(stream) if stream else None))
        return nodes, lengths

    def close(self):
        if self._h is not None and self._h.value:
            L.lib().mhw_session_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_count() -> int:
    return L.lib().mhw_device_count()
