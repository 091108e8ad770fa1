"""Parity at BASELINE.json's full sizes.

* The cfg2 / cfg3 / cfg4 graphs the bench walks (device R-MAT / hetero
  generators + device build_csr) equal the oracle's generators + build_csr
  array for array, and their graph_checksum (FNV-1a of tools/mhwalk.cpp:
  107-122) matches -- the reference's own loader semantics are pinned to the
  oracle's build_csr in test_oracle_vs_reference.py / test_loader.py.
* Static alias tables of the cfg1 and cfg4 graphs equal alias_build
  (samplers.cpp:95-131) node by node, bit for bit.
* Per-step decisions on the cfg2 / cfg3 / cfg4 graphs: 1M random (state,
  candidate, last, u) triples per model, plus adversarial u = wc/wl +- 1 ulp,
  equal the oracle's calculate_weight + accept bit for bit.
* cfg5 (R-MAT scale 26, 2.1G arcs; too large for the host oracle): the
  size-independent CSR properties -- verified symmetric, sorted duplicate-free
  self-loop-free slices, degree sum = arcs.
* A cfg2 walk partition (the bench's session config, one 1/16 node range):
  every transition is an arc of the graph, rows start at their node, lengths
  are L+1 except at isolated starts, and the stats add up.
The oracle runs on the host here (a few minutes in total)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import model_desc, random_triples, walk_model

pytestmark = pytest.mark.gpu

SEED = 1  # bench.py SEED


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


@pytest.fixture(scope="module")
def cfg2(mhw, oracle):
    dg = mhw.Graph.rmat(20, 16, seed=SEED)
    lo, hi = oracle.rmat_pairs(20, 16, seed=SEED)
    return dg, oracle.build_csr(lo, hi, None, symmetrize=True, n_nodes=1 << 20)


@pytest.fixture(scope="module")
def cfg4(mhw, oracle):
    dg = mhw.Graph.rmat(22, 16, seed=SEED, weighted=True, weight_lo=1.0, weight_hi=10.0, edge_types=4)
    lo, hi = oracle.rmat_pairs(22, 16, seed=SEED)
    w = oracle.pair_weights(SEED, lo, hi, 1.0, 10.0).astype(np.float64)
    hg = oracle.build_csr(lo, hi, w, symmetrize=True, n_nodes=1 << 22)
    src = np.repeat(np.arange(hg.n, dtype=np.uint32), np.diff(hg.offsets).astype(np.int64))
    hg.etype = oracle.pair_etypes(SEED, np.minimum(src, hg.nbr), np.maximum(src, hg.nbr), 4)
    hg.n_etypes = 4
    return dg, hg


@pytest.fixture(scope="module")
def cfg3(mhw, oracle):
    n = 2_000_000
    dg = mhw.Graph.hetero(n, seed=SEED, weight_lo=1.0, weight_hi=5.0)
    lo, hi, nA, nP = oracle.hetero_pairs(n, seed=SEED)
    w = oracle.pair_weights(SEED, lo, hi, 1.0, 5.0).astype(np.float64)
    hg = oracle.build_csr(lo, hi, w, symmetrize=True, n_nodes=n)
    hg.ntype = np.zeros(n, dtype=np.uint16)
    hg.ntype[nA:nA + nP] = 1
    hg.ntype[nA + nP:] = 2
    hg.n_ntypes = 3
    return dg, hg


def _check_csr(oracle, d, hg, weighted):
    assert np.array_equal(d["offsets"].astype(np.uint64), hg.offsets)
    assert np.array_equal(d["neighbors"].astype(np.uint32), hg.nbr)
    w_dev = d["weights"].astype(np.float64) if weighted else None
    if weighted:
        assert np.array_equal(w_dev, hg.w)
    assert oracle.graph_checksum(d["offsets"], d["neighbors"], w_dev) == \
        oracle.graph_checksum(hg.offsets, hg.nbr, hg.w if weighted else None)


def test_cfg2_graph_fullsize(oracle, cfg2):
    """R-MAT scale 20, edge factor 16, unweighted (cfg2)."""
    dg, hg = cfg2
    _check_csr(oracle, dg.download(), hg, weighted=False)
    assert hg.m == 31_402_114


def test_cfg4_graph_fullsize(oracle, cfg4):
    """R-MAT scale 22, fp32 U[1,10) per undirected edge, 4 edge types (cfg4)."""
    dg, hg = cfg4
    d = dg.download()
    _check_csr(oracle, d, hg, weighted=True)
    assert np.array_equal(d["edge_types"], hg.etype)


def test_cfg3_graph_fullsize(oracle, cfg3):
    """A/P/V hetero graph, 2M nodes, fp32 U[1,5) (cfg3a / cfg3b)."""
    dg, hg = cfg3
    d = dg.download()
    _check_csr(oracle, d, hg, weighted=True)
    assert np.array_equal(d["node_types"], hg.ntype)


def test_cfg1_cfg4_alias_tables_fullsize(mhw, oracle, cfg4):
    g1 = mhw.Graph.rmat(16, 16, seed=SEED, weighted=True, weight_lo=1.0, weight_hi=10.0)
    d = g1.download()
    for dg, off, w in ((g1, d["offsets"], d["weights"].astype(np.float64)), (cfg4[0], cfg4[1].offsets, cfg4[1].w)):
        prob, alias = mhw.alias_tables(dg)
        oprob, oalias = oracle.alias_tables(off, w)
        assert np.array_equal(prob.view(np.uint64), oprob.view(np.uint64))
        assert np.array_equal(alias, oalias)


def _decide_parity(mhw, oracle, dg, hg, md, n=1_000_000, seed=0):
    pos, aff, cand, last, u = random_triples(hg, md, n, seed=seed)
    ow = oracle.decide(hg, md, pos, aff, cand, last, u)
    gw = mhw.decide(dg, walk_model(md), pos, aff, cand, last, u)
    for a, b in zip(ow, gw):
        assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
    # adversarial: u at wc/wl and one ulp either side
    wc, wl = ow[0], ow[1]
    ok = wl > 0
    r = (wc[ok] / wl[ok])
    for uu in (r, np.nextafter(r, 0), np.nextafter(r, 1)):
        uu = np.clip(uu, 0.0, np.nextafter(1.0, 0))
        args = (pos[ok], aff[ok], cand[ok], last[ok], uu)
        assert np.array_equal(oracle.decide(hg, md, *args)[2], mhw.decide(dg, walk_model(md), *args)[2])


def test_cfg2_decisions_fullsize(mhw, oracle, cfg2):
    dg, hg = cfg2
    _decide_parity(mhw, oracle, dg, hg, model_desc(O.NODE2VEC, hg, p=0.25, q=4.0), seed=2)


def test_cfg4_decisions_fullsize(mhw, oracle, cfg4):
    import bench
    dg, hg = cfg4
    dg.set_node_types(np.zeros(hg.n, dtype=np.uint16), 1)
    hg.ntype, hg.n_ntypes = np.zeros(hg.n, dtype=np.uint16), 1
    cfg = dict(bench.CONFIGS["cfg4"])
    md = model_desc(O.EDGE2VEC, hg, p=cfg["p"], q=cfg["q"], M=bench.type_matrix(cfg))
    _decide_parity(mhw, oracle, dg, hg, md, seed=4)


def test_cfg3_decisions_fullsize(mhw, oracle, cfg3):
    dg, hg = cfg3
    for kind, seed in ((O.METAPATH2VEC, 31), (O.FAIRWALK, 32)):
        md = model_desc(kind, hg, p=1.0, q=1.0, metapath=(0, 1, 2, 1, 0))
        _decide_parity(mhw, oracle, dg, hg, md, n=500_000, seed=seed)


def test_cfg5_graph_properties(mhw):
    """R-MAT scale 26 (cfg5): the device CSR is symmetric (every arc has its
    back arc), slices are sorted, duplicate- and self-loop-free, degrees sum
    to the arc count."""
    dg = mhw.Graph.rmat(26, 16, seed=SEED)
    d = dg.download()
    # binding a second-order model builds the reverse-arc index, which
    # verifies that every arc has its back arc
    v = int(np.argmax(np.diff(d["offsets"])))
    m = mhw.WalkModel(kind=mhw.ModelKind.node2vec, p=0.25, q=4.0)
    mhw.decide(dg, m, [v], [0], [0], [1], [0.5])
    info = dg.info()
    assert info["verified_symmetric"] == 1
    off = d["offsets"].astype(np.int64)
    nb = d["neighbors"]
    assert off[0] == 0 and off[-1] == len(nb) == info["arc_count"] > 2_000_000_000
    deg = np.diff(off)
    assert (deg >= 0).all()
    rng = np.random.default_rng(5)
    for v in np.concatenate([rng.choice(np.nonzero(deg)[0], 200_000, replace=False),
                             np.argsort(deg)[-200:]]):
        s = nb[off[v]:off[v + 1]]
        assert (np.diff(s.astype(np.int64)) > 0).all() and not (s == v).any(), v


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
