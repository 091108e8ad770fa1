"""Parity at BASELINE.json's full sizes.

* The cfg2 / cfg3 / cfg4 graphs the bench walks (device R-MAT / hetero
  generators + device build_csr) equal the oracle's generators + build_csr
  array for array, and their graph_checksum (FNV-1a of tools/mhwalk.cpp:
  107-122) matches -- the reference's own loader semantics are pinned to the
  oracle's build_csr in test_oracle_vs_reference.py / test_loader.py.
* A cfg2 walk partition (the bench's session config, one 1/16 node range):
  size-independent properties -- every transition is an arc of the graph,
  rows start at their node, lengths are L+1 except at isolated starts, and
  the stats add up.
The oracle runs on the host here (about a minute at scale 22)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEED = 1  # bench.py SEED


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def _check_csr(oracle, d, hg, weighted):
    assert np.array_equal(d["offsets"].astype(np.uint64), hg.offsets)
    assert np.array_equal(d["neighbors"].astype(np.uint32), hg.nbr)
    w_dev = d["weights"].astype(np.float64) if weighted else None
    if weighted:
        assert np.array_equal(w_dev, hg.w)
    assert oracle.graph_checksum(d["offsets"], d["neighbors"], w_dev) == \
        oracle.graph_checksum(hg.offsets, hg.nbr, hg.w if weighted else None)


def test_cfg2_graph_fullsize(mhw, oracle):
    """R-MAT scale 20, edge factor 16, unweighted (cfg2)."""
    dg = mhw.Graph.rmat(20, 16, seed=SEED)
    lo, hi = oracle.rmat_pairs(20, 16, seed=SEED)
    hg = oracle.build_csr(lo, hi, None, symmetrize=True, n_nodes=1 << 20)
    _check_csr(oracle, dg.download(), hg, weighted=False)
    assert hg.m == 31_402_114


def test_cfg4_graph_fullsize(mhw, oracle):
    """R-MAT scale 22, fp32 U[1,10) per undirected edge, 4 edge types (cfg4)."""
    dg = mhw.Graph.rmat(22, 16, seed=SEED, weighted=True, weight_lo=1.0, weight_hi=10.0, edge_types=4)
    lo, hi = oracle.rmat_pairs(22, 16, seed=SEED)
    w = oracle.pair_weights(SEED, lo, hi, 1.0, 10.0).astype(np.float64)
    hg = oracle.build_csr(lo, hi, w, symmetrize=True, n_nodes=1 << 22)
    d = dg.download()
    _check_csr(oracle, d, hg, weighted=True)
    src = np.repeat(np.arange(hg.n, dtype=np.uint32), np.diff(hg.offsets).astype(np.int64))
    a, b = np.minimum(src, hg.nbr), np.maximum(src, hg.nbr)
    assert np.array_equal(d["edge_types"], oracle.pair_etypes(SEED, a, b, 4))


def test_cfg3_graph_fullsize(mhw, oracle):
    """A/P/V hetero graph, 2M nodes, fp32 U[1,5) (cfg3a / cfg3b)."""
    n = 2_000_000
    dg = mhw.Graph.hetero(n, seed=SEED, weight_lo=1.0, weight_hi=5.0)
    lo, hi, nA, nP = oracle.hetero_pairs(n, seed=SEED)
    w = oracle.pair_weights(SEED, lo, hi, 1.0, 5.0).astype(np.float64)
    hg = oracle.build_csr(lo, hi, w, symmetrize=True, n_nodes=n)
    d = dg.download()
    _check_csr(oracle, d, hg, weighted=True)
    t = d["node_types"]
    assert (t[:nA] == 0).all() and (t[nA:nA + nP] == 1).all() and (t[nA + nP:] == 2).all()


def test_cfg2_walk_partition_properties(mhw):
    import bench
    cfg = dict(bench.CONFIGS["cfg2"])
    cfg["name"] = "cfg2"
    g = bench.build_graph(cfg)
    model = bench.make_model(cfg)
    n = g.node_count()
    b, e = 7 * n // 16, 8 * n // 16
    c = mhw.generate_walks(g, model, bench.make_config(cfg, b, e))
    d = g.download()
    off = d["offsets"].astype(np.int64)
    nbr = d["neighbors"].astype(np.uint64)
    deg = np.diff(off)
    starts = np.repeat(np.arange(b, e), cfg["K"])
    rows, lens = c.rows, c.lengths
    assert len(lens) == (e - b) * cfg["K"] == c.stats.walks
    assert np.array_equal(rows[:, 0].astype(np.int64), starts)
    iso = deg[starts] == 0
    assert (lens[iso] == 1).all() and (lens[~iso] == cfg["L"] + 1).all()
    assert c.stats.steps == int((lens.astype(np.int64) - 1).sum())
    assert c.stats.early_terminations == int(iso.sum())
    # every transition is an arc: keys (src << 32 | dst) of the CSR are sorted
    src = np.repeat(np.arange(n, dtype=np.uint64), deg)
    keys = (src << np.uint64(32)) | nbr
    full = rows[~iso][:, :cfg["L"] + 1].astype(np.uint64)
    q = ((full[:, :-1] << np.uint64(32)) | full[:, 1:]).ravel()
    pos = np.searchsorted(keys, q)
    assert (pos < len(keys)).all() and np.array_equal(keys[np.minimum(pos, len(keys) - 1)], q)
