"""The benchmarked throughput kernel (k_walk) pinned bit for bit at BASELINE
scale.

Every headline number comes from k_walk (walk.cu), whose decision code --
narrow 8-byte records with the speculative Last fetch, the pre-issued edge
filter probe, fairwalk's pre-read group sizes, the w'(Last) cached in typed
records, hub replicas -- is not the code of the parity kernels (k_decide,
k_det_*). A walker that runs ALONE is deterministic on the throughput
schedule (nobody else touches its chains), so each of ~2000 starts per config
(the top-degree hubs plus random starts) is walked alone through
mhw_session_select_starts (K = 1, the bench's graph, model, init strategy and
kernel variant, eagerly initialised tables installed before each run where
the bench initialises eagerly) and compared byte for byte with the oracle's
og_walk_isolated: the same walker with a fresh SamplerManager
(manager.cpp:30-72), walker-major (engine.cpp:178-205), Philox layout.
Reference: test_engine.cpp:116-124 (single-thread determinism).
"""
import dataclasses
import os

import numpy as np
import pytest

import bench
from oracle import oracle as O

pytestmark = pytest.mark.gpu

N_HUBS = 150
N_RANDOM = 1850
KIND = {"deepwalk": O.DEEPWALK, "node2vec": O.NODE2VEC, "metapath2vec": O.METAPATH2VEC,
        "edge2vec": O.EDGE2VEC, "fairwalk": O.FAIRWALK}


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def host_graph(dg):
    """The device CSR as the oracle's host graph (the device CSR itself is
    pinned to the oracle's generators + build_csr in test_gpu_fullsize.py)."""
    d = dg.download()
    m = len(d["neighbors"])
    w = d["weights"].astype(np.float64) if d["weights"] is not None else np.ones(m)
    return O.HostGraph(d["offsets"].astype(np.uint64), d["neighbors"].astype(np.uint32), w,
                       ntype=d["node_types"], etype=d["edge_types"], n_ntypes=d["num_node_types"],
                       n_etypes=d["num_edge_types"], symmetric=True)


def oracle_model(cfg):
    md = O.ModelDesc(kind=KIND[cfg["model"]], p=cfg["p"], q=cfg["q"])
    if cfg["model"] == "metapath2vec":
        md.metapath = list(cfg["metapath"])
    if cfg["model"] == "edge2vec":
        md.type_matrix = bench.type_matrix(cfg)
    return md


def oracle_cfg(cfg, K, replica_degree, proposal=0):
    init = {"random": O.INIT_RANDOM, "high_weight": O.INIT_HIGH_WEIGHT, "burn_in": O.INIT_BURN_IN}[cfg["init"]]
    return O.WalkCfg(K=K, L=cfg["L"], seed=bench.WALK_SEED, init_kind=init, burn_in_steps=cfg.get("burn_in", 100),
                     hw_sample_size=32, replica_degree=replica_degree, proposal=proposal)


def pick_starts(hg, cfg, seed):
    deg = np.diff(hg.offsets.astype(np.int64))
    ok = deg > 0
    if cfg["model"] == "metapath2vec":
        ok &= hg.ntype == cfg["metapath"][0]
    cand = np.nonzero(ok)[0]
    hubs = cand[np.argsort(-deg[cand], kind="stable")[:N_HUBS]]
    rest = np.setdiff1d(cand, hubs)
    r = np.random.default_rng(seed)
    rnd = r.choice(rest, size=min(N_RANDOM, len(rest)), replace=False)
    return np.sort(np.concatenate([hubs, rnd])).astype(np.uint32)


def pin(mhw, oracle, cfg_name, init_mode=0, env=None, n_starts=None, proposal=0):
    cfg = dict(bench.CONFIGS[cfg_name])
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        dg = bench.build_graph(cfg)
        wc = dataclasses.replace(bench.make_config(cfg), walks_per_node=1, init_mode=init_mode, proposal=proposal)
        s = mhw.Session(dg, bench.make_model(cfg), wc)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    hg = host_graph(dg)
    md = oracle_model(cfg)
    starts = pick_starts(hg, cfg, seed=len(cfg_name) + init_mode)
    if n_starts:
        starts = starts[:: max(1, len(starts) // n_starts)]
    # eagerly initialised second-order sessions: install the initial table
    # before every single-walker run (the bench's LAZY = false kernel variant)
    table = None
    second = cfg["model"] in ("node2vec", "edge2vec", "fairwalk")
    if second and init_mode == 2:
        import torch
        table = torch.empty(s.chain_size() * s.record_width(), dtype=torch.int32, device="cuda")
        s.init_records(0, s.chain_size(), table.data_ptr())
        torch.cuda.synchronize()
    orows, olens, ost = oracle.walk_isolated(hg, md, oracle_cfg(cfg, 1, wc.chain_replica_degree, proposal), starts)
    assert len(olens) == len(starts)
    steps = 0
    for j, v in enumerate(starts):
        # the first 100 eager runs initialise the table themselves (the bench's
        # k_init_all / k_init_rec launch), the rest install the saved table
        if table is not None and j >= 100:
            s.load_records(table.data_ptr())
        s.select_starts([int(v)])
        s.run()
        st = s.stats()
        rows, lens = s.download()
        assert lens[0] == olens[j], (cfg_name, int(v), int(lens[0]), int(olens[j]))
        assert np.array_equal(rows[0, :lens[0]], orows[j, :olens[j]]), (cfg_name, int(v))
        assert st.chain_retries == 0
        if table is not None and j >= 100:
            assert st.slot_inits == 0
        steps += int(lens[0]) - 1
    s.close()
    return len(starts), steps


@pytest.mark.parametrize("cfg_name", ["cfg1", "cfg3a"])
def test_kwalk_node_keyed_single_walkers_equal_oracle(mhw, oracle, cfg_name):
    """deepwalk (graph arc records, automatic hub replicas, lazy init) and
    metapath2vec (typed session records, visit-weighted replicas, typed-index
    slot init) on the full cfg1 / cfg3 graphs."""
    n, steps = pin(mhw, oracle, cfg_name)
    assert n >= 1500 and steps > 50 * n


@pytest.mark.parametrize("cfg_name", ["cfg2", "cfg3b", "cfg4"])
def test_kwalk_second_order_single_walkers_equal_oracle(mhw, oracle, cfg_name):
    """node2vec (narrow records, speculative Last fetch, pre-issued edge
    filter probe, L2-pinned filter, burn-in init), fairwalk (typed records,
    pre-read group sizes, cached w'(Last)) and edge2vec (typed records, 2-bit
    L2 filter, cached w'(Last)) on the full graphs, eager tables (the bench's
    variant), plus lazy first-touch init on a subset."""
    n, steps = pin(mhw, oracle, cfg_name, init_mode=2)
    assert n >= 1500 and steps > 50 * n
    pin(mhw, oracle, cfg_name, init_mode=1, n_starts=300)


def test_kwalk_wide_records_equal_oracle(mhw, oracle):
    """The cfg5 kernel variant on the cfg2 graph: 16-byte node2vec records
    {u, deg, off, chain word} and random init in record order (k_init_rec),
    with an 8-bit-per-arc edge filter (cfg5's density)."""
    env = {"MHW_C16": "0", "MHW_NARROW": "0", "MHW_BLOOM_BITS": "8"}
    cfg = dict(bench.CONFIGS["cfg2"], init="random")
    bench.CONFIGS["cfg2_wide"] = cfg
    try:
        pin(mhw, oracle, "cfg2_wide", init_mode=2, env=env, n_starts=800)
    finally:
        del bench.CONFIGS["cfg2_wide"]


@pytest.mark.parametrize("layout,env", [
    ("narrow", {"MHW_C16": "0", "MHW_NARROW": "1"}),
    ("c16_pin_both", {"MHW_C16": "1", "MHW_C16_PIN": "both"}),
])
def test_kwalk_cfg2_chain_layouts_equal_oracle(mhw, oracle, layout, env):
    """cfg2 with the other node2vec chain layouts: the narrow {u, chain word}
    records (round-1 kernel) and the compact 16-bit table pinned in L2 with
    a copy of the edge filter. The default (compact table, filter pinned) is
    test_kwalk_second_order_single_walkers_equal_oracle[cfg2]; its hub
    states (degree >= 2^14: cfg2's top hubs) keep no alpha class in the
    16-bit word, which the 150 hub starts exercise."""
    n, steps = pin(mhw, oracle, "cfg2", init_mode=2, env=env, n_starts=800)
    assert n >= 700 and steps > 50 * n


def _hub_graph(hub_deg=20000, seed=5):
    """An unweighted hub of degree >= 2^14 (compact chain words of its states
    hold no alpha class) inside a ring of leaves with random chords, so that
    candidates of every alpha class occur at the hub."""
    r = np.random.default_rng(seed)
    n = hub_deg + 1
    pairs = {(0, i) for i in range(1, n)}
    pairs |= {(min(i, i % hub_deg + 1), max(i, i % hub_deg + 1)) for i in range(1, n)}
    a = r.integers(1, n, 3 * hub_deg)
    b = r.integers(1, n, 3 * hub_deg)
    pairs |= {(int(min(x, y)), int(max(x, y))) for x, y in zip(a, b) if x != y}
    edges = [(x, y, 1.0) for x, y in pairs] + [(y, x, 1.0) for x, y in pairs]  # symmetric, no duplicates
    return O.make_graph(n, edges, symmetric=True)


def test_kwalk_compact_hub_states_equal_oracle(mhw, oracle):
    """Compact chains at a hub of degree 20,000 (>= 2^14): the walker
    recomputes the Last's alpha class from its id; single walkers equal the
    oracle byte for byte."""
    import os as _os
    from tests.helpers import device_graph, model_desc, walk_config
    g = _hub_graph()
    md = model_desc(O.NODE2VEC, g, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=1, L=40, seed=11, init_kind=O.INIT_BURN_IN, burn_in_steps=10)
    old = _os.environ.get("MHW_C16")
    _os.environ["MHW_C16"] = "1"
    try:
        dg = device_graph(g, weighted=False)
        s = mhw.Session(dg, mhw.WalkModel(kind=mhw.ModelKind.node2vec, p=0.25, q=4.0),
                        walk_config(cfg, threads=8, init_mode=2))
    finally:
        if old is None:
            _os.environ.pop("MHW_C16", None)
        else:
            _os.environ["MHW_C16"] = old
    assert s.shard_entry_bytes() == 2  # compact chains are in use
    starts = np.concatenate([[0], np.arange(1, g.n, 97)]).astype(np.uint32)
    orows, olens, _ = oracle.walk_isolated(g, md, cfg, starts)
    hub_visits = 0
    for j, v in enumerate(starts):
        s.select_starts([int(v)])
        s.run()
        rows, lens = s.download()
        assert lens[0] == olens[j] and np.array_equal(rows[0, :lens[0]], orows[j, :olens[j]]), int(v)
        hub_visits += int(np.sum(rows[0, 1:lens[0]] == 0))
    assert hub_visits > 100  # the hub states were walked through
    s.close()


def test_compact_hub_states_pass_chain_chi_square(mhw, oracle):
    """Throughput corpus on the hub graph with compact chains: the hub states
    (x, 0) (degree 20,000: the word holds no class, recomputed every step)
    pass the lumped chain chi-square. Their return class is one candidate in
    20,000, so a valid test needs ~10^5 transitions per state (min_entries):
    2,000,000 walkers of 2 steps from each of 5 leaves, all arriving at the
    hub at once (the lock protocol under its heaviest contention)."""
    import os as _os
    from tests.helpers import device_graph, model_desc, walk_config
    from tests.stats import audit_counts, gate, transition_counts_gpu
    g = _hub_graph()
    md = model_desc(O.NODE2VEC, g, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=2_000_000, L=2, seed=13, init_kind=O.INIT_BURN_IN, burn_in_steps=10)
    old = _os.environ.get("MHW_C16")
    _os.environ["MHW_C16"] = "1"
    try:
        c = mhw.generate_walks(device_graph(g, weighted=False),
                               mhw.WalkModel(kind=mhw.ModelKind.node2vec, p=0.25, q=4.0),
                               walk_config(cfg, threads=8, init_mode=2, node_begin=1, node_end=6))
    finally:
        if old is None:
            _os.environ.pop("MHW_C16", None)
        else:
            _os.environ["MHW_C16"] = old
    assert c.stats.chain_retries > 0
    states = transition_counts_gpu(c.rows, c.lengths, O.NODE2VEC, g.offsets, g.nbr, min_visits=100_000,
                                   max_states=80)
    hub = [st for st in states if st[0] == 0]
    assert len(hub) == 5, [(st[0], st[2]) for st in states]
    pv = audit_counts(g, oracle, md, hub, min_entries=5)
    assert len(pv) == 5
    ok, msg = gate(pv)
    assert ok, msg
