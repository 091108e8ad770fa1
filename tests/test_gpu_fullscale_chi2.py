"""The north star's distribution gate on BASELINE-scale throughput corpora.

Walk-level transition frequencies per state against the exact normalised
w' (tools/mhwalk.cpp:208-220), with the Markov-chain CLT chi-square of
tests/stats.py, on the benchmarked kernel (k_walk) and the BASELINE graphs:

* cfg1 (deepwalk, R-MAT s16) and cfg3a (metapath2vec, 2M-node hetero graph):
  the bench's full corpus (K = 10); cfg1's states with >= 5000 visits and
  <= 1024 neighbours, cfg3a's venue (V) states.
* cfg2 (node2vec), cfg3b (fairwalk), cfg4 (edge2vec): a second-order state
  (s, v) is visited ~16-80 times in a K = 10 run (steps / arcs), so K is
  raised on one start node s of degree >= 32 (the adjacency hash-set branch
  of the alpha test) until its states (s, v) and the return states (v, s)
  reach >= 5000 visits; every walker passes them, so their chains are also
  the most contended ones (the lock protocol under load). For unweighted
  node2vec the test lumps candidates of equal target weight (exact for the
  uniform-proposal kernel), so hub states of any degree are audited too.

Per-state p-values go through the family gate (gate(): Bonferroni floor,
Fisher, and the count of p < 0.01 against chance). Transition counting runs
on the GPU with torch (test infrastructure only).
Reference: test_engine.cpp:136-163 (pooled next-node frequencies at states
with >= 5000 visits).
"""
import dataclasses

import numpy as np
import pytest

import bench
from oracle import oracle as O
from tests.stats import audit_counts, gate, transition_counts_gpu
from tests.test_gpu_kwalk_pin import KIND, host_graph, oracle_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def run_corpus(mhw, dg, cfg, **over):
    wc = dataclasses.replace(bench.make_config(cfg), **over)
    s = mhw.Session(dg, bench.make_model(cfg), wc)
    s.run()
    st = s.stats()
    rows, lens = s.download()
    s.close()
    return rows, lens, st


def check(mhw, oracle, cfg_name, hg, rows, lens, max_support, min_states=20, max_states=40):
    cfg = bench.CONFIGS[cfg_name]
    md = oracle_model(cfg)
    states = transition_counts_gpu(rows, lens, KIND[cfg["model"]], hg.offsets, hg.nbr,
                                   metapath=cfg.get("metapath"), min_visits=5000, max_states=max_states,
                                   max_support=max_support)
    assert len(states) >= min_states, f"{cfg_name}: only {len(states)} states with >= 5000 visits"
    pv = audit_counts(hg, oracle, md, states, min_entries=5)
    assert len(pv) >= min_states // 2, f"{cfg_name}: only {len(pv)} of {len(states)} states are valid for the test"
    ok, msg = gate(pv)
    assert ok, f"{cfg_name}: {msg}"
    return states, pv


@pytest.mark.parametrize("cfg_name", ["cfg1", "cfg3a"])
def test_full_corpus_chain_chi_square(mhw, oracle, cfg_name):
    cfg = bench.CONFIGS[cfg_name]
    dg = bench.build_graph(cfg)
    hg = host_graph(dg)
    rows, lens, st = run_corpus(mhw, dg, cfg)
    assert st.steps == int(np.sum(lens.astype(np.int64) - 1))
    states, pv = check(mhw, oracle, cfg_name, hg, rows, lens, max_support=1024)
    if cfg_name == "cfg3a":  # the venue states (type V) are the hot ones
        assert sum(hg.ntype[v] == 2 for v, *_ in states) >= 10


def pick_start(hg, cfg, lo, hi, max_support, need=None):
    """A start of degree in [lo, hi] with the most neighbours of degree <=
    max_support (weighted graphs: the audited states (s, v) need a dense
    test), at least `need` of them (R-MAT neighbours are mostly hubs)."""
    deg = np.diff(hg.offsets.astype(np.int64))
    cands = np.nonzero((deg >= lo) & (deg <= hi))[0]
    r = np.random.default_rng(3)
    best, best_n = None, -1
    for v in r.permutation(cands)[:4000]:
        nb = hg.neighbors_of(int(v)).astype(np.int64)
        k = int(np.sum(deg[nb] <= max_support))
        if k > best_n:
            best, best_n = int(v), k
        if k >= 0.9 * len(nb):
            break
    need = lo if need is None else need
    assert best_n >= need, f"no start node found (best has {best_n} light neighbours)"
    return best


@pytest.mark.parametrize("cfg_name,deg_lo,deg_hi,max_support,walkers_per_arc", [
    ("cfg2", 40, 60, None, 7000),     # unweighted node2vec: lumped test at any degree
    ("cfg3b", 18, 30, 1024, 20000),   # fairwalk from a P node (A and V neighbours)
    ("cfg4", 32, 40, 1024, 16000),    # edge2vec, weighted bootstrap
])
def test_hub_start_chain_chi_square(mhw, oracle, cfg_name, deg_lo, deg_hi, max_support, walkers_per_arc):
    cfg = bench.CONFIGS[cfg_name]
    dg = bench.build_graph(cfg)
    hg = host_graph(dg)
    s0 = pick_start(hg, cfg, deg_lo, deg_hi, max_support or 1 << 30)
    K = walkers_per_arc * hg.degree(s0)
    # eager tables: the bench's kernel variant for these configs
    rows, lens, st = run_corpus(mhw, dg, cfg, walks_per_node=K, node_begin=s0, node_end=s0 + 1, init_mode=2)
    assert len(lens) == K and np.all(rows[:, 0] == s0)
    assert st.chain_retries > 0  # the step-1 states are contended by design
    check(mhw, oracle, cfg_name, hg, rows, lens, max_support=max_support)
