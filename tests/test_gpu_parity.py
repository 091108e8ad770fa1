"""GPU parity against the CPU oracle (the C restatement pinned to the
reference, see test_oracle_vs_reference.py). Everything here calls the CUDA
kernels through the C ABI (libmhw.so)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import (INITS, KINDS, corpus_equal, device_graph, model_desc, random_triples,
                           typed_random_graph, walk_config, walk_model)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0, "no CUDA device: the engine has no CPU fallback"
    return m


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("weighted", [True, False])
def test_decide_bit_exact(mhw, oracle, kind, weighted):
    """Per-step decisions on identical (state, cand, last, u) triples are
    bit-exact (samplers.hpp:21-26, models.cpp:82-123)."""
    g = typed_random_graph(31 + kind, 300, 6.0, weighted=weighted, types=3)
    md = model_desc(kind, g, p=0.37, q=1.9, metapath=(0, 1, 2, 1, 0),
                    M=np.random.default_rng(5).uniform(0.5, 2.0, (9, 9)))
    dg = device_graph(g, weighted)
    pos, aff, cand, last, u = random_triples(g, md, 20000, seed=kind)
    owc, owl, oacc = oracle.decide(g, md, pos, aff, cand, last, u)
    # adversarial unit draws exactly at the decision boundary (u = wc/wl +- 1 ulp)
    ratio = np.where(owl > 0, owc / np.where(owl > 0, owl, 1), 0.5)
    k = len(u) // 4
    u[:k] = np.clip(ratio[:k], 0, np.nextafter(1, 0))
    u[k:2 * k] = np.clip(np.nextafter(ratio[k:2 * k], 2), 0, np.nextafter(1, 0))
    u[2 * k:3 * k] = np.clip(np.nextafter(ratio[2 * k:3 * k], -1), 0, np.nextafter(1, 0))
    owc, owl, oacc = oracle.decide(g, md, pos, aff, cand, last, u)
    gwc, gwl, gacc = mhw.decide(dg, walk_model(md), pos, aff, cand, last, u)
    assert np.array_equal(owc.view(np.uint64), gwc.view(np.uint64))
    assert np.array_equal(owl.view(np.uint64), gwl.view(np.uint64))
    assert np.array_equal(oacc, gacc)


def rmat_host(oracle, scale=11, seed=9, types=3):
    lo, hi = oracle.rmat_pairs(scale, 16, seed=seed)
    w = oracle.pair_weights(seed, lo, hi, 1.0, 10.0).astype(np.float64)
    hg = oracle.build_csr(lo, hi, w, symmetrize=True, n_nodes=1 << scale)
    hg.ntype = np.random.default_rng(seed).integers(0, types, hg.n).astype(np.uint16)
    hg.n_ntypes = types
    return hg


@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_decide_bit_exact_on_hubs(mhw, oracle, kind):
    """Hub-heavy R-MAT graph: alpha goes through the adjacency hash sets
    (degree >= 32) and the shorter-slice search; decisions stay bit-exact."""
    hg = rmat_host(oracle)
    assert np.diff(hg.offsets).max() >= 256
    md = model_desc(kind, hg, p=0.4, q=2.5, M=np.random.default_rng(2).uniform(0.5, 2.0, (9, 9)))
    pos, aff, cand, last, u = random_triples(hg, md, 50000, seed=kind)
    # bias half of the states onto the top hubs
    deg = np.diff(hg.offsets).astype(np.int64)
    hubs = np.argsort(deg)[-32:]
    pos[::2] = hubs[np.arange(len(pos[::2])) % 32]
    d = deg[pos]
    cand, last = cand % d, last % d
    aff = np.where(aff == O.NO_AFFIX, aff, aff % d)
    owc, owl, oacc = oracle.decide(hg, md, pos, aff, cand, last, u)
    gwc, gwl, gacc = mhw.decide(device_graph(hg), walk_model(md), pos, aff, cand, last, u)
    assert np.array_equal(owc.view(np.uint64), gwc.view(np.uint64))
    assert np.array_equal(owl.view(np.uint64), gwl.view(np.uint64))
    assert np.array_equal(oacc, gacc)


@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_deterministic_walks_on_hubs_equal_oracle(mhw, oracle, kind):
    hg = rmat_host(oracle, scale=10, seed=4)
    md = model_desc(kind, hg, p=0.25, q=4.0, M=np.random.default_rng(3).uniform(0.5, 2.0, (9, 9)))
    cfg = O.WalkCfg(K=2, L=40, seed=8, init_kind=O.INIT_BURN_IN, burn_in_steps=10)
    orow, olen, _ = oracle.generate_walks(hg, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    corpus = mhw.generate_walks(device_graph(hg), walk_model(md), walk_config(cfg))
    assert corpus_equal(orow, olen, corpus.rows, corpus.lengths)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("init", INITS)
def test_deterministic_walks_equal_oracle(mhw, oracle, kind, init):
    """The deterministic schedule reproduces the oracle's (philox, step-major)
    corpus byte for byte: bootstrap, lazy slot init, M-H chain, update_state."""
    g = typed_random_graph(7 + kind, 120, 5.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=4, L=25, seed=99 + init, init_kind=init, burn_in_steps=10, hw_sample_size=4)
    orow, olen, ost = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    dg = device_graph(g)
    corpus = mhw.generate_walks(dg, walk_model(md), walk_config(cfg, threads=1))
    assert corpus_equal(orow, olen, corpus.rows, corpus.lengths)
    s = corpus.stats
    assert (s.walks, s.early_terminations, s.skipped_starts, s.steps) == (
        ost["walks"], ost["early_terminations"], ost["skipped_starts"], ost["steps"])


@pytest.mark.parametrize("kind", [O.DEEPWALK, O.METAPATH2VEC])
@pytest.mark.parametrize("rep", [0, 1, 4, 16])
def test_deterministic_hub_replicas_equal_oracle(mhw, oracle, kind, rep):
    """Node-keyed chains replicated at hubs (degree >= rep): same layout and
    walker->replica map on both sides, corpus byte-identical."""
    rng = O.XoRng(21)
    g = O.preferential_attachment(300, 3, rng)
    O.assign_random_types(g, 2, rng)
    g.w = np.array([float(np.float32(0.5 + rng.uniform_real())) for _ in range(g.m)])
    # symmetric weights are not needed for first-order models
    md = model_desc(kind, g)
    cfg = O.WalkCfg(K=6, L=30, seed=3, init_kind=O.INIT_BURN_IN, burn_in_steps=5, replica_degree=rep)
    orow, olen, ost = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    corpus = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg))
    assert corpus_equal(orow, olen, corpus.rows, corpus.lengths)
    assert corpus.stats.slot_inits == ost["init_calls"]


@pytest.mark.parametrize("kind", KINDS)
def test_deterministic_unweighted_and_isolated(mhw, oracle, kind):
    """Unweighted graph (bootstrap closed form) with isolated nodes."""
    rng = O.XoRng(3)
    g = O.random_graph(60, 3.0, False, rng, ensure_connected=False)
    O.assign_random_types(g, 2, rng)
    md = model_desc(kind, g, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=3, L=30, seed=5, init_kind=O.INIT_BURN_IN, burn_in_steps=10)
    orow, olen, ost = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    corpus = mhw.generate_walks(device_graph(g, weighted=False), walk_model(md), walk_config(cfg))
    assert corpus_equal(orow, olen, corpus.rows, corpus.lengths)
    assert corpus.stats.early_terminations == ost["early_terminations"]


@pytest.mark.parametrize("kind", KINDS)
def test_throughput_walks_valid(mhw, kind):
    """Throughput schedule: corpus shape/order, edge validity, metapath
    compliance (test_engine.cpp:64-114, acceptance.cpp:266-288)."""
    g = typed_random_graph(11 + kind, 400, 8.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.5, q=2.0)
    cfg = O.WalkCfg(K=5, L=40, seed=17, init_kind=O.INIT_RANDOM)
    corpus = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=8))
    n_valid = g.n if kind != O.METAPATH2VEC else int(np.sum(g.ntype == md.metapath[0]))
    assert len(corpus) == n_valid * cfg.K
    assert corpus.stats.skipped_starts == (g.n - n_valid) * cfg.K
    adj = set()
    for v in range(g.n):
        for u in g.neighbors_of(v):
            adj.add((v, int(u)))
    starts = [v for v in range(g.n) if kind != O.METAPATH2VEC or g.ntype[v] == md.metapath[0]]
    for r, walk in enumerate(corpus.walks):
        assert walk[0] == starts[r // cfg.K]
        for a, b in zip(walk[:-1], walk[1:]):
            assert (int(a), int(b)) in adj
        if kind == O.METAPATH2VEC:
            for i, x in enumerate(walk):
                assert g.ntype[x] == (0 if i % 2 == 0 else 1)
    assert corpus.stats.steps == int(np.sum(corpus.lengths - 1))


def test_packed_corpus_equals_padded(mhw, oracle):
    """mhw_generate_walks_packed (device compaction + D2H) == the padded corpus."""
    from paper_2010_04895_b200.mhwalk import generate_walks_packed
    g = typed_random_graph(61, 150, 5.0, weighted=True, types=2)
    rng = O.XoRng(1)
    md = model_desc(O.NODE2VEC, g, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=3, L=30, seed=5, init_kind=O.INIT_BURN_IN, burn_in_steps=10)
    dg = device_graph(g)
    padded = mhw.generate_walks(dg, walk_model(md), walk_config(cfg, threads=1))
    nodes, offsets, st = generate_walks_packed(dg, walk_model(md), walk_config(cfg, threads=1))
    assert len(offsets) == len(padded) + 1
    assert np.array_equal(np.diff(offsets), padded.lengths)
    for r in range(len(padded)):
        assert np.array_equal(nodes[offsets[r]:offsets[r + 1]], padded.rows[r, :padded.lengths[r]])
    assert st.steps == padded.stats.steps
    assert rng is not None


@pytest.mark.parametrize("kind", KINDS)
def test_check_audit_equals_oracle(mhw, oracle, kind):
    """`check` (tools/mhwalk.cpp:222-247) on the GPU: per-state chain visit
    counts identical to og_check, KL within 1e-12, and below the reference's
    chain-correctness bound (acceptance.cpp:44-63: KL < 0.005 at 1e6 draws)."""
    g = typed_random_graph(71 + kind, 200, 8.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.4, q=2.5)
    pos, aff, _, _, _ = random_triples(g, md, 64, seed=kind)
    if kind in (O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK):
        deg = np.diff(g.offsets).astype(np.int64)[pos]
        aff = np.where(aff == O.NO_AFFIX, 0, aff) % deg
    if kind == O.METAPATH2VEC:  # states must have the metapath position's type
        keep = g.ntype[pos] == np.array(md.metapath)[aff]
        pos, aff = pos[keep], aff[keep]
    okl, ocnt = oracle.check(g, md, 99, pos, aff, 100000)
    from paper_2010_04895_b200.mhwalk import check
    gkl, gcnt, code = check(device_graph(g), walk_model(md), pos, aff, 100000, seed=99, tolerance=0.005)
    assert np.array_equal(ocnt, gcnt)
    both = ~np.isnan(okl)
    assert np.array_equal(both, ~np.isnan(gkl))
    assert np.allclose(okl[both], gkl[both], rtol=1e-12, atol=1e-15)
    assert code == 0


@pytest.mark.parametrize("kind", [O.DEEPWALK, O.NODE2VEC, O.METAPATH2VEC])
def test_packed_overlapped_throughput_corpus(mhw, kind):
    """Throughput schedule through the chunked walk + overlapped D2H path:
    corpus order, start nodes, edge validity, lengths and step count."""
    from paper_2010_04895_b200.mhwalk import generate_walks_packed
    g = typed_random_graph(81 + kind, 3000, 6.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.5, q=2.0)
    cfg = O.WalkCfg(K=4, L=25, seed=3)
    nodes, offsets, st = generate_walks_packed(device_graph(g), walk_model(md), walk_config(cfg, threads=8))
    starts = [v for v in range(g.n) if kind != O.METAPATH2VEC or g.ntype[v] == md.metapath[0]]
    assert len(offsets) == len(starts) * cfg.K + 1
    lens = np.diff(offsets.astype(np.int64))
    assert lens.min() >= 1 and lens.max() <= cfg.L + 1
    assert st.steps == int(np.sum(lens - 1))
    adj = {(v, int(u)) for v in range(g.n) for u in g.neighbors_of(v)}
    for r in range(len(lens)):
        w = nodes[offsets[r]:offsets[r + 1]]
        assert w[0] == starts[r // cfg.K]
        assert all((int(a), int(b)) in adj for a, b in zip(w[:-1], w[1:]))


def test_alias_tables_bit_exact(mhw, oracle):
    """Per-node alias tables == alias_build (samplers.cpp:95-131) bit for bit."""
    g = typed_random_graph(41, 500, 10.0, weighted=True)
    prob, alias = mhw.alias_tables(device_graph(g))
    for v in range(g.n):
        w = g.weights_of(v)
        if len(w) == 0:
            continue
        op, oa = oracle.alias_build(w)
        a, b = g.offsets[v], g.offsets[v + 1]
        assert np.array_equal(op.view(np.uint64), prob[a:b].view(np.uint64)), v
        assert np.array_equal(oa, alias[a:b]), v


@pytest.mark.parametrize("scale,weighted,etypes", [(10, True, 0), (12, False, 4), (16, True, 0)])
def test_rmat_csr_bit_exact(mhw, oracle, scale, weighted, etypes):
    """Device R-MAT generator + CSR build == oracle generator + build_csr."""
    lo, hi = oracle.rmat_pairs(scale, 16, seed=7)
    w = oracle.pair_weights(7, lo, hi, 1.0, 10.0).astype(np.float64) if weighted else None
    hg = oracle.build_csr(lo, hi, w, symmetrize=True, n_nodes=1 << scale)
    dg = mhw.Graph.rmat(scale, 16, seed=7, weighted=weighted, weight_lo=1.0, weight_hi=10.0, edge_types=etypes)
    d = dg.download()
    assert np.array_equal(d["offsets"].astype(np.uint64), hg.offsets)
    assert np.array_equal(d["neighbors"].astype(np.uint32), hg.nbr)
    if weighted:
        assert np.array_equal(d["weights"].astype(np.float64), hg.w)
    if etypes:
        src = np.repeat(np.arange(hg.n), np.diff(hg.offsets).astype(np.int64))
        a, b = np.minimum(src, hg.nbr), np.maximum(src, hg.nbr)
        assert np.array_equal(d["edge_types"], oracle.pair_etypes(7, a, b, etypes))


def test_hetero_csr_bit_exact(mhw, oracle):
    lo, hi, nA, nP = oracle.hetero_pairs(5000, seed=3)
    w = oracle.pair_weights(3, lo, hi, 1.0, 5.0).astype(np.float64)
    hg = oracle.build_csr(lo, hi, w, symmetrize=True, n_nodes=5000)
    d = mhw.Graph.hetero(5000, seed=3).download()
    assert np.array_equal(d["offsets"].astype(np.uint64), hg.offsets)
    assert np.array_equal(d["neighbors"].astype(np.uint32), hg.nbr)
    assert np.array_equal(d["weights"].astype(np.float64), hg.w)
    t = d["node_types"]
    assert (t[:nA] == 0).all() and (t[nA:nA + nP] == 1).all() and (t[nA + nP:] == 2).all()


def test_from_edges_build_csr_semantics(mhw, oracle):
    """build_csr (graph.cpp:35-66): sort, duplicate sum, symmetrize without
    self-loop doubling, n = max id + 1."""
    r = np.random.default_rng(0)
    src = r.integers(0, 50, 400)
    dst = r.integers(0, 50, 400)
    w = r.integers(1, 8, 400).astype(np.float32) / 4  # dyadic: sums exact in any order
    hg = oracle.build_csr(src, dst, w.astype(np.float64), symmetrize=True)
    d = mhw.Graph.from_edges(src, dst, w, symmetrize=True).download()
    assert np.array_equal(d["offsets"].astype(np.uint64), hg.offsets)
    assert np.array_equal(d["neighbors"].astype(np.uint32), hg.nbr)
    assert np.array_equal(d["weights"].astype(np.float64), hg.w)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("init", INITS)
def test_slot_init_equals_oracle(mhw, oracle, kind, init):
    """mh_init (samplers.cpp:37-83) under the slot-keyed Philox layout."""
    g = typed_random_graph(51 + kind, 200, 12.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.3, q=3.0)
    cfg = O.WalkCfg(K=1, L=1, seed=1234, init_kind=init, burn_in_steps=13, hw_sample_size=5)
    pos, aff, _, _, _ = random_triples(g, md, 400, seed=kind * 3 + init)
    if kind in (O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK):
        deg = np.diff(g.offsets).astype(np.int64)[pos]
        aff = np.where(aff == O.NO_AFFIX, 0, aff) % deg
    got = mhw.init_states(device_graph(g), walk_model(md), walk_config(cfg), pos, aff)
    gs, ms, keep = oracle.bind(g, md)
    for i in range(len(pos)):
        v, a = int(pos[i]), int(aff[i])
        if kind == O.DEEPWALK:
            slot = v
        elif kind == O.METAPATH2VEC:
            mp = md.metapath
            nxt = a + 1 if a + 1 < len(mp) else (1 if mp[0] == mp[-1] and len(mp) > 1 else 0)
            slot = v * g.n_ntypes + mp[nxt]
        else:
            slot = int(g.offsets[v]) + a
        want = oracle.init_philox(g, md, cfg, v, a, slot)
        assert (O.NO_AFFIX if want is None else want) == got[i], (i, v, a)


@pytest.mark.parametrize("init", [O.INIT_RANDOM, O.INIT_HIGH_WEIGHT, O.INIT_BURN_IN])
def test_metapath_typed_index_init_equals_scan(mhw, oracle, init):
    """metapath2vec slot inits pick the pick-th positive (required type, w > 0)
    through the typed neighbour index; the oracle scans the slice
    (samplers.cpp:22-33). Zero weights, three types, hubs of degree > 32."""
    rng = O.XoRng(77)
    g = O.random_graph(300, 24.0, True, rng)
    O.assign_random_types(g, 3, rng)
    r = np.random.default_rng(5)
    w = g.w.copy()
    zero = r.uniform(size=g.m) < 0.25
    w[zero] = 0.0
    g.w = w
    md = model_desc(O.METAPATH2VEC, g, metapath=(0, 1, 2, 1, 0))
    cfg = O.WalkCfg(K=1, L=1, seed=99, init_kind=init, burn_in_steps=7, hw_sample_size=4)
    n = g.n
    pos = np.repeat(np.arange(n, dtype=np.uint32), 5)
    aff = np.tile(np.arange(5, dtype=np.uint32), n)
    got = mhw.init_states(device_graph(g), walk_model(md), walk_config(cfg), pos, aff)
    mp = md.metapath
    for i in range(len(pos)):
        v, a = int(pos[i]), int(aff[i])
        nxt = a + 1 if a + 1 < len(mp) else (1 if mp[0] == mp[-1] else 0)
        want = oracle.init_philox(g, md, cfg, v, a, v * g.n_ntypes + mp[nxt])
        assert (O.NO_AFFIX if want is None else want) == got[i], (i, v, a)


@pytest.mark.parametrize("bits", ["2", "8", "0"])
@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC])
def test_decide_bit_exact_any_edge_filter_density(mhw, oracle, kind, bits, monkeypatch):
    """The edge filter only ever short-cuts to 'not adjacent' on a miss: the
    alpha classes, hence the decisions, are the same at every density the
    build policy picks (2 bits/arc L2-resident, 8 bits/arc DRAM-resident) and
    without a filter (MHW_BLOOM=0)."""
    if bits == "0":
        monkeypatch.setenv("MHW_BLOOM", "0")
    else:
        monkeypatch.setenv("MHW_BLOOM_BITS", bits)
    rng = O.XoRng(700 + kind)
    g = O.preferential_attachment(600, 6, rng)  # hubs: hash sets and long slices
    O.assign_random_types(g, 2, rng)
    g.w = np.array([float(np.float32(0.5 + rng.uniform_real())) for _ in range(g.m)])
    md = model_desc(kind, g, p=0.37, q=1.9)
    dg = device_graph(g)
    pos, aff, cand, last, u = random_triples(g, md, 20000, seed=kind + 11)
    owc, owl, oacc = oracle.decide(g, md, pos, aff, cand, last, u)
    gwc, gwl, gacc = mhw.decide(dg, walk_model(md), pos, aff, cand, last, u)
    assert np.array_equal(owc.view(np.uint64), gwc.view(np.uint64))
    assert np.array_equal(owl.view(np.uint64), gwl.view(np.uint64))
    assert np.array_equal(oacc, gacc)
