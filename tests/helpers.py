"""Shared builders for the parity tests: one model spec -> oracle ModelDesc and
engine WalkModel, graphs built the way the reference's tests build them
(tests/oracles.hpp:27-118, restated in oracle/oracle.py)."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O

KINDS = [O.DEEPWALK, O.NODE2VEC, O.METAPATH2VEC, O.EDGE2VEC, O.FAIRWALK]
INITS = [O.INIT_RANDOM, O.INIT_HIGH_WEIGHT, O.INIT_BURN_IN]


def model_desc(kind, g: O.HostGraph, p=0.5, q=2.0, metapath=(0, 1, 0), M=None) -> O.ModelDesc:
    md = O.ModelDesc(kind=kind, p=p, q=q)
    if kind == O.METAPATH2VEC:
        md.metapath = list(metapath)
    if kind == O.EDGE2VEC:
        dim = g.n_etypes if g.etype is not None else g.n_ntypes * g.n_ntypes
        md.type_matrix = np.ones((dim, dim)) if M is None else np.asarray(M, dtype=np.float64)
    return md


def walk_model(md: O.ModelDesc):
    from paper_2010_04895_b200 import ModelKind, WalkModel
    return WalkModel(kind=ModelKind(md.kind), p=md.p, q=md.q, metapath=list(md.metapath),
                     type_matrix=md.type_matrix)


def walk_config(cfg: O.WalkCfg, threads=1, **kw):
    from paper_2010_04895_b200 import InitKind, InitStrategy, SamplerKind, WalkConfig
    kw.setdefault("chain_replica_degree", cfg.replica_degree)
    kw.setdefault("sampler_kind", SamplerKind(cfg.sampler))
    return WalkConfig(walks_per_node=cfg.K, walk_length=cfg.L, threads=threads, seed=cfg.seed,
                      init=InitStrategy(InitKind(cfg.init_kind), cfg.burn_in_steps, cfg.hw_sample_size), **kw)


def typed_random_graph(seed, n, avg_deg, weighted=True, types=2) -> O.HostGraph:
    rng = O.XoRng(seed)
    g = O.random_graph(n, avg_deg, weighted, rng)
    O.assign_random_types(g, types, rng)
    return g


def device_graph(g: O.HostGraph, weighted=True):
    from paper_2010_04895_b200 import Graph
    return Graph.from_host(g, weighted=weighted)


def random_triples(g: O.HostGraph, md: O.ModelDesc, count, seed):
    """Random (state, cand, last, u) triples over valid states of the model,
    like tools/mhwalk.cpp:183-206 draws audit states."""
    r = np.random.default_rng(seed)
    deg = np.diff(g.offsets).astype(np.int64)
    nz = np.nonzero(deg)[0]
    pos = r.choice(nz, size=count)
    d = deg[pos]
    cand = (r.random(count) * d).astype(np.int64)
    last = (r.random(count) * d).astype(np.int64)
    if md.kind == O.METAPATH2VEC:
        aff = r.integers(0, len(md.metapath), size=count)
    elif md.kind in (O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK):
        aff = (r.random(count) * d).astype(np.int64)
        boot = r.random(count) < 0.1
        aff[boot] = O.NO_AFFIX
    else:
        aff = np.full(count, O.NO_AFFIX)
    u = r.random(count)
    return pos, aff, cand, last, u


def corpus_equal(rows_a, lens_a, rows_b, lens_b):
    if len(lens_a) != len(lens_b) or not np.array_equal(lens_a, lens_b):
        return False
    for i in range(len(lens_a)):
        if not np.array_equal(rows_a[i, :lens_a[i]], rows_b[i, :lens_b[i]]):
            return False
    return True
