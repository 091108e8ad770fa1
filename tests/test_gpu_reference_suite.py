"""The reference's own engine / model / sampler tests (proj/tests/*.cpp and
acceptance.cpp), restated against the GPU engine through the Python mirror of
the mhwalk API, plus the north-star chi-square gate on throughput-mode
corpora. Graph builders restate tests/oracles.hpp (oracle/oracle.py)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import device_graph, model_desc, typed_random_graph, walk_config, walk_model
from tests.stats import audit, gate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def bound(mhw, kind, g, p=1.0, q=1.0):
    md = model_desc(kind, g, p=p, q=q)
    return md, walk_model(md)


def valid(g, corpus):
    adj = {(v, int(u)) for v in range(g.n) for u in g.neighbors_of(v)}
    return all((int(a), int(b)) in adj for w in corpus.walks for a, b in zip(w[:-1], w[1:]))


# ------------------------------------------------------------ test_engine.cpp
@pytest.mark.parametrize("threads", [1, 8])
def test_isolated_node_emits_length1_walks(mhw, threads):            # :40-48
    g = O.make_graph(1, [])
    c = mhw.generate_walks(device_graph(g), walk_model(model_desc(O.DEEPWALK, g)),
                           mhw.WalkConfig(walks_per_node=2, walk_length=80, threads=threads))
    assert len(c) == 2 and all(list(w) == [0] for w in c.walks)
    assert c.stats.early_terminations == 2


def test_triangle_full_length_valid_walks(mhw):                       # :50-62
    g = O.triangle()
    c = mhw.generate_walks(device_graph(g), walk_model(model_desc(O.DEEPWALK, g)),
                           mhw.WalkConfig(walks_per_node=1, walk_length=3, seed=9))
    assert len(c) == 3 and all(len(w) == 4 for w in c.walks)
    assert valid(g, c)
    assert [int(w[0]) for w in c.walks] == [0, 1, 2]


def test_walk_count_is_nodes_minus_skipped_times_K(mhw):             # :64-74
    rng = O.XoRng(1)
    g = O.random_graph(60, 5.0, False, rng)
    O.assign_random_types(g, 2, rng)
    c = mhw.generate_walks(device_graph(g, False), walk_model(model_desc(O.METAPATH2VEC, g)),
                           mhw.WalkConfig(walks_per_node=3, walk_length=10, seed=2))
    assert len(c) == g.n * 3 - c.stats.skipped_starts
    assert c.stats.skipped_starts > 0


@pytest.mark.parametrize("threads", [1, 8])
def test_every_model_emits_edge_valid_walks(mhw, threads):          # :76-86
    rng = O.XoRng(3)
    g = O.random_graph(80, 6.0, True, rng)
    O.assign_random_types(g, 2, rng)
    dg = device_graph(g)
    for kind in range(5):
        c = mhw.generate_walks(dg, walk_model(model_desc(kind, g, 0.5, 2.0)),
                               mhw.WalkConfig(walks_per_node=2, walk_length=20, seed=4, threads=threads))
        assert valid(g, c)


def test_every_sampler_kind_emits_edge_valid_walks(mhw):              # :88-98
    rng = O.XoRng(5)
    g = O.random_graph(60, 5.0, True, rng)
    dg = device_graph(g)
    for kind in mhw.SamplerKind:
        c = mhw.generate_walks(dg, walk_model(model_desc(O.NODE2VEC, g, 0.5, 2.0)),
                               mhw.WalkConfig(walks_per_node=2, walk_length=15, seed=6, sampler_kind=kind))
        assert len(c) == 120 and valid(g, c)


@pytest.mark.parametrize("threads", [1, 8])
def test_metapath_walks_follow_metapath_cyclically(mhw, threads):    # :100-114
    rng = O.XoRng(7)
    g = O.random_graph(80, 8.0, False, rng)
    O.assign_random_types(g, 2, rng)
    c = mhw.generate_walks(device_graph(g, False), walk_model(model_desc(O.METAPATH2VEC, g)),
                           mhw.WalkConfig(walks_per_node=3, walk_length=20, seed=8, threads=threads))
    assert len(c) > 0
    for w in c.walks:
        assert all(g.ntype[x] == (0 if i % 2 == 0 else 1) for i, x in enumerate(w))


def test_single_threaded_seeded_runs_are_identical(mhw, tmp_path):  # :116-124, acceptance 8
    rng = O.XoRng(9)
    g = O.random_graph(100, 5.0, True, rng)
    dg, m = device_graph(g), walk_model(model_desc(O.NODE2VEC, g, 0.25, 4.0))
    cfg = mhw.WalkConfig(walks_per_node=2, walk_length=30, threads=1, seed=1234)
    a, b = mhw.generate_walks(dg, m, cfg), mhw.generate_walks(dg, m, cfg)
    assert a.walks.__len__() == b.walks.__len__()
    assert np.array_equal(a.rows, b.rows) and np.array_equal(a.lengths, b.lengths)
    pa, pb = str(tmp_path / "a.txt"), str(tmp_path / "b.txt")
    mhw.write_corpus(a, pa)
    mhw.write_corpus(b, pb)
    assert open(pa, "rb").read() == open(pb, "rb").read()


def test_multithreaded_runs_count(mhw):                               # :126-134
    rng = O.XoRng(10)
    g = O.random_graph(100, 5.0, False, rng)
    c = mhw.generate_walks(device_graph(g, False), walk_model(model_desc(O.DEEPWALK, g)),
                           mhw.WalkConfig(walks_per_node=4, walk_length=20, threads=4, seed=11))
    assert len(c) == 400 and valid(g, c)


@pytest.mark.parametrize("threads", [1, 8])
def test_pooled_next_node_frequencies(mhw, oracle, threads):          # :136-163
    rng = O.XoRng(12)
    g = O.preferential_attachment(50, 3, rng)
    c = mhw.generate_walks(device_graph(g), walk_model(model_desc(O.DEEPWALK, g)),
                           mhw.WalkConfig(walks_per_node=50, walk_length=80, seed=13, threads=threads))
    trans = np.zeros((g.n, g.n))
    for w in c.walks:
        for a, b in zip(w[:-1], w[1:]):
            trans[a, b] += 1
    audited = 0
    for v in range(g.n):
        visits = trans[v].sum()
        if visits < 5000:
            continue
        audited += 1
        target = g.weights_of(v) / g.weights_of(v).sum()
        freq = trans[v, g.neighbors_of(v)] / visits
        assert np.abs(freq - target).max() < 0.05
    assert audited > 0


def test_second_half_closer_than_first_half(mhw, oracle):            # :165-201
    rng = O.XoRng(14)
    g = O.random_graph(12, 5.0, True, rng)
    dg, m = device_graph(g), walk_model(model_desc(O.DEEPWALK, g))
    kl = np.zeros(2)
    for seed in range(20):
        c = mhw.generate_walks(dg, m, mhw.WalkConfig(walks_per_node=20, walk_length=80, seed=seed))
        for half in (0, 1):
            tot, acc = 0, 0.0
            for v in range(g.n):
                counts = np.zeros(g.degree(v))
                for w in c.walks:
                    lo, hi = (len(w) // 2, len(w)) if half else (1, len(w) // 2)
                    for i in range(lo, hi):
                        if w[i - 1] == v:
                            counts[np.searchsorted(g.neighbors_of(v), w[i])] += 1
                n = counts.sum()
                if n == 0:
                    continue
                p = counts[counts > 0] / n
                t = (g.weights_of(v) / g.weights_of(v).sum())[counts > 0]
                acc += n * float(np.sum(p * np.log(p / t)))
                tot += n
            kl[half] += acc / tot
    assert kl[1] < kl[0]


# ------------------------------------------------------------ test_models.cpp
def dec(mhw, g, md, pos, aff, cand, last=None):
    n = len(pos)
    return mhw.decide(device_graph(g), walk_model(md), pos, aff, cand, cand if last is None else last, np.zeros(n))


def test_model_known_answers(mhw):                                   # :46-106
    g = O.make_graph(2, [(0, 1, 2.5), (1, 0, 2.5)])
    assert dec(mhw, g, model_desc(O.DEEPWALK, g), [0], [O.NO_AFFIX], [0])[0][0] == 2.5
    tri = O.triangle()
    back = int(np.searchsorted(tri.neighbors_of(1), 0))
    wc = dec(mhw, tri, model_desc(O.NODE2VEC, tri, p=0.25, q=1.0), [1], [0], [back])[0][0]
    assert wc == 4.0
    t = O.triangle()
    t.ntype, t.n_ntypes = np.array([0, 1, 1], dtype=np.uint16), 2
    md = model_desc(O.METAPATH2VEC, t)
    wc = dec(mhw, t, md, [0, 0], [0, 0], [0, 1])[0]
    assert list(wc) == [1.0, 1.0]
    wc = dec(mhw, t, md, [1], [1], [int(np.searchsorted(t.neighbors_of(1), 2))])[0]
    assert wc[0] == 0.0
    f = O.make_graph(5, [(0, 1, 1), (0, 2, 1), (0, 3, 1), (0, 4, 1), (1, 0, 1), (2, 0, 1), (3, 0, 1), (4, 0, 1)])
    f.ntype, f.n_ntypes = np.array([0, 0, 0, 1, 1], dtype=np.uint16), 2
    wc = dec(mhw, f, model_desc(O.FAIRWALK, f, p=1.0, q=1.0), [0] * 4, [0] * 4, [0, 1, 2, 3])[0]
    assert np.allclose(wc, 0.5)


def test_node2vec_p_q_1_is_deepwalk(mhw):                            # :52-65
    rng = O.XoRng(5)
    g = O.random_graph(40, 5.0, True, rng)
    pos, aff, cand = [], [], []
    for v in range(g.n):
        for s in range(g.degree(v)):
            for i in range(g.degree(v)):
                pos.append(v), aff.append(s), cand.append(i)
    a = dec(mhw, g, model_desc(O.NODE2VEC, g, p=1.0, q=1.0), pos, aff, cand)[0]
    b = dec(mhw, g, model_desc(O.DEEPWALK, g), pos, [O.NO_AFFIX] * len(pos), cand)[0]
    assert np.array_equal(a, b)


def test_normalised_weights_match_equation_oracles(mhw, oracle):    # :209-256, acceptance 7
    rng = O.XoRng(101)
    for trial in range(3):
        g = O.random_graph(30 + 30 * trial, 6.0, True, rng)
        O.assign_random_types(g, 3, rng)
        p, q = 0.25 + rng.uniform_real(), 0.25 + 2 * rng.uniform_real()
        dg = device_graph(g)
        for kind in (O.NODE2VEC, O.FAIRWALK):
            md = model_desc(kind, g, p, q)
            for v in range(g.n):
                d = g.degree(v)
                for s in range(d):
                    wc = mhw.decide(dg, walk_model(md), [v] * d, [s] * d, range(d), range(d), np.zeros(d))[0]
                    got = wc / wc.sum()
                    prev = g.neighbors_of(v)[s]
                    nb = g.neighbors_of(v)
                    alpha = np.array([1 / p if u == prev else (1.0 if u in set(g.neighbors_of(prev)) else 1 / q)
                                      for u in nb])
                    w = alpha * g.weights_of(v)
                    if kind == O.FAIRWALK:
                        grp = np.array([np.sum(g.ntype[nb] == g.ntype[u]) for u in nb])
                        w = w / grp
                    assert np.abs(got - w / w.sum()).max() < 1e-12


def test_bind_rejections(mhw):                                       # :194-207
    g = O.make_graph(2, [(0, 1, 1.0)], symmetric=False)
    with pytest.raises(mhw.ValidationError, match="symmetric"):
        mhw.generate_walks(device_graph(g), walk_model(model_desc(O.NODE2VEC, g)), mhw.WalkConfig())
    t = O.triangle()
    with pytest.raises(mhw.ValidationError, match="node types"):
        mhw.generate_walks(device_graph(t), mhw.WalkModel(kind=mhw.ModelKind.metapath2vec, metapath=[0, 1]),
                           mhw.WalkConfig())


# ---------------------------------------------------------- test_samplers.cpp
def hub(weights):
    edges = []
    for i, w in enumerate(weights):
        edges += [(0, i + 1, float(w)), (i + 1, 0, float(w))]
    return O.make_graph(len(weights) + 1, edges)


def init_of(mhw, g, md, kind, seed=1, burn=100, hw=32, state=(0, O.NO_AFFIX)):
    cfg = O.WalkCfg(K=1, L=1, seed=seed, init_kind=kind, burn_in_steps=burn, hw_sample_size=hw)
    return int(mhw.init_states(device_graph(g), walk_model(md), walk_config(cfg), [state[0]], [state[1]])[0])


def test_high_weight_init(mhw):                                       # :34-50
    g = hub([1, 1, 9])
    assert init_of(mhw, g, model_desc(O.DEEPWALK, g), O.INIT_HIGH_WEIGHT) == 2
    g = hub([3, 3, 3, 1])
    assert init_of(mhw, g, model_desc(O.DEEPWALK, g), O.INIT_HIGH_WEIGHT) == 0


def test_random_init_uniform_over_positive(mhw):                      # :52-67
    g = hub([1, 0, 1, 0, 1])
    md = model_desc(O.DEEPWALK, g)
    cfg = O.WalkCfg(K=1, L=1, init_kind=O.INIT_RANDOM)
    dg, m = device_graph(g), walk_model(md)
    counts = np.zeros(5)
    for seed in range(3000):
        cfg.seed = seed
        counts[int(mhw.init_states(dg, m, walk_config(cfg), [0], [O.NO_AFFIX])[0])] += 1
    assert counts[1] == 0 and counts[3] == 0
    assert np.abs(counts[[0, 2, 4]] / 3000 - 1 / 3).max() < 0.04


def test_dead_end_init(mhw):                                          # :69-78, test_manager :120-127
    g = hub([0, 0])
    for kind in O.INIT_RANDOM, O.INIT_HIGH_WEIGHT, O.INIT_BURN_IN:
        assert init_of(mhw, g, model_desc(O.DEEPWALK, g), kind) == O.NO_AFFIX
    c = mhw.generate_walks(device_graph(g), walk_model(model_desc(O.DEEPWALK, g)),
                           mhw.WalkConfig(walks_per_node=2, walk_length=5, threads=8))
    assert all(len(w) == 1 for w in c.walks) and c.stats.early_terminations == len(c)


def test_burn_in_lands_on_positive(mhw):                              # :80-90
    g = hub([0, 2, 5, 0, 1])
    for seed in range(50):
        last = init_of(mhw, g, model_desc(O.DEEPWALK, g), O.INIT_BURN_IN, seed=seed)
        assert g.weights_of(0)[last] > 0


def test_restricted_support_init(mhw):                                # :92-112
    g = hub([1, 1, 1, 1, 1])
    g.ntype, g.n_ntypes = np.array([0, 1, 0, 0, 1, 0], dtype=np.uint16), 2
    md = model_desc(O.METAPATH2VEC, g, metapath=(0, 1))
    for seed in range(40):
        for kind in O.INIT_RANDOM, O.INIT_HIGH_WEIGHT, O.INIT_BURN_IN:
            assert init_of(mhw, g, md, kind, seed=seed, state=(0, 0)) in (0, 3)


# ---------------------------------------------------------- acceptance.cpp 8
def test_acceptance_walk_validity(mhw):                              # :266-304
    rng = O.XoRng(1008)
    g = O.random_graph(1000, 8.0, True, rng)
    O.assign_random_types(g, 2, rng)
    dg = device_graph(g)
    for threads in (1, 8):
        cfg = mhw.WalkConfig(walks_per_node=10, walk_length=40, threads=threads, seed=1008)
        c = mhw.generate_walks(dg, walk_model(model_desc(O.NODE2VEC, g, 0.5, 2.0)), cfg)
        assert len(c) == 10000 and valid(g, c)
        t = mhw.generate_walks(dg, walk_model(model_desc(O.METAPATH2VEC, g)), cfg)
        for w in t.walks:
            assert all(g.ntype[x] == (0 if i % 2 == 0 else 1) for i, x in enumerate(w))


# ------------------------------------------------- north star: chi-square gate
@pytest.mark.parametrize("kind", [O.DEEPWALK, O.NODE2VEC, O.METAPATH2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_throughput_transitions_pass_chain_chi_square(mhw, oracle, kind):
    """Per-state transition frequencies of the throughput schedule vs the exact
    normalised w' (Markov-chain chi-square, tests/stats.py), states with >=
    5000 visits; the same audit on the CPU oracle corpus is the control."""
    g = typed_random_graph(300 + kind, 40, 4.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.5, q=2.0, M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)))
    cfg = O.WalkCfg(K=400, L=80, seed=77, init_kind=O.INIT_RANDOM)
    c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=8))
    pv = audit(g, oracle, md, c.rows, c.lengths, min_visits=5000)
    ok, msg = gate(pv)
    assert ok, msg
    rows, lens, _ = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    ok_c, msg_c = gate(audit(g, oracle, md, rows, lens, min_visits=5000))
    assert ok_c, "control: " + msg_c


LAYOUTS = {  # node2vec chain-word layouts of the throughput kernel
    "wide": {"MHW_C16": "0", "MHW_NARROW": "0"},    # 16-byte {u, deg, off, chain word} records
    "narrow": {"MHW_C16": "0", "MHW_NARROW": "1"},  # 8-byte {u, chain word} records
    "c16": {"MHW_C16": "1"},                        # ids + compact 16-bit chain table (eager only)
    "c16_pin_both": {"MHW_C16": "1", "MHW_C16_PIN": "both"},  # [c16 | filter copy] in one L2 window
    "c16_pin_chain": {"MHW_C16": "1", "MHW_C16_PIN": "chain"},
}


@pytest.mark.parametrize("layout", sorted(LAYOUTS))
def test_node2vec_record_layouts_pass_chain_chi_square(mhw, oracle, layout, monkeypatch):
    """node2vec chain layouts: 16-byte {u, deg, off, chain word} records, the
    narrow 8-byte {u, chain word} layout (node record from L2) and the
    compact 16-bit chain table beside the plain ids (eager init only; lazy
    runs fall back to records), eager and lazy slot init."""
    for k, v in LAYOUTS[layout].items():
        monkeypatch.setenv(k, v)
    g = typed_random_graph(901, 40, 4.0, weighted=False, types=2)
    md = model_desc(O.NODE2VEC, g, p=0.25, q=4.0)
    # burn-in: eager init in slot order; random init on wide records: eager
    # init in record order (the cfg5 path)
    for init_mode, init_kind in ((1, O.INIT_BURN_IN), (2, O.INIT_BURN_IN), (2, O.INIT_RANDOM)):
        cfg = O.WalkCfg(K=400, L=80, seed=79 + init_mode + init_kind, init_kind=init_kind, burn_in_steps=4)
        c = mhw.generate_walks(device_graph(g, weighted=False), walk_model(md),
                               walk_config(cfg, threads=8, init_mode=init_mode))
        ok, msg = gate(audit(g, oracle, md, c.rows, c.lengths, min_visits=5000))
        assert ok, msg


@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_lazy_colocated_chains_pass_chain_chi_square(mhw, oracle, kind):
    """Second-order throughput walks with lazy slot init (init_mode 1): the
    colocated chain words start EMPTY and are initialised on first visit with
    the slot-keyed draws; explicit edge types for edge2vec."""
    g = typed_random_graph(500 + kind, 40, 4.0, weighted=True, types=2)
    r = np.random.default_rng(kind)
    pairs = {}
    for v in range(g.n):
        for u in g.neighbors_of(v):
            pairs.setdefault((min(v, int(u)), max(v, int(u))), int(r.integers(0, 3)))
    g.etype = np.array([pairs[(min(v, int(u)), max(v, int(u)))] for v in range(g.n) for u in g.neighbors_of(v)],
                       dtype=np.uint16)
    g.n_etypes = 3
    md = model_desc(kind, g, p=0.5, q=2.0, M=r.uniform(0.5, 2.0, (3, 3)))
    cfg = O.WalkCfg(K=400, L=80, seed=78, init_kind=O.INIT_BURN_IN, burn_in_steps=3)
    c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=8, init_mode=1))
    ok, msg = gate(audit(g, oracle, md, c.rows, c.lengths, min_visits=5000))
    assert ok, msg


@pytest.mark.parametrize("rep", [8, 1, 0])
def test_hub_replicas_pass_chain_chi_square(mhw, oracle, rep):
    """Deepwalk on a hub-heavy graph with replicated hub chains (8, every
    node (1), and the automatic layout (0))."""
    rng = O.XoRng(12)
    g = O.preferential_attachment(60, 3, rng)
    md = model_desc(O.DEEPWALK, g)
    cfg = O.WalkCfg(K=300, L=80, seed=5, replica_degree=rep)
    c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=8))
    ok, msg = gate(audit(g, oracle, md, c.rows, c.lengths, min_visits=5000))
    assert ok, msg


# ------------------------------------------------------------- partitioning
def test_partition_and_multi_replica_corpus(mhw):
    """mhw_partition_nodes == the host rule; generate_walks_multi over two
    replicas concatenates shards in the reference corpus order."""
    from paper_2010_04895_b200.partition import balanced_cuts
    dg = mhw.Graph.rmat(12, 16, seed=3)
    d = dg.download()
    deg = np.diff(d["offsets"])
    model = mhw.WalkModel(kind=mhw.ModelKind.node2vec, p=0.25, q=4.0)
    for parts in (1, 2, 3, 8):
        assert np.array_equal(mhw.partition_nodes(dg, model, parts), balanced_cuts(deg, parts))
    rep = dg.replicate(0)
    cfg = mhw.WalkConfig(walks_per_node=2, walk_length=10, threads=8, seed=1)
    multi = mhw.generate_walks_multi([dg, rep], model, cfg)
    single = mhw.generate_walks(dg, model, cfg)
    assert len(multi) == len(single)
    assert np.array_equal(multi.rows[:, 0], single.rows[:, 0])
    assert multi.stats.steps == int(np.sum(multi.lengths - 1))
