"""Edge cases of the walk path on the GPU: empty and tiny graphs, walk
length 1, start-node ranges, dead ends, asymmetric adjacency behind a
symmetric flag (update_state's error, models.cpp:131-133), and the
one-chain-per-state layout switch."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import corpus_equal, device_graph, model_desc, typed_random_graph, walk_config, walk_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def test_empty_graph(mhw):
    g = mhw.Graph.from_csr(np.array([0]), np.array([], dtype=np.int32))
    assert g.node_count() == 0 and g.arc_count() == 0
    for threads in (1, 8):
        c = mhw.generate_walks(g, mhw.WalkModel(), mhw.WalkConfig(threads=threads))
        assert len(c) == 0 and c.stats.steps == 0


def test_walk_length_one_and_single_walk(mhw, oracle):
    g = typed_random_graph(5, 50, 4.0)
    for kind in range(5):
        md = model_desc(kind, g)
        cfg = O.WalkCfg(K=1, L=1, seed=3)
        orow, olen, _ = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
        c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg))
        assert corpus_equal(orow, olen, c.rows, c.lengths)
        assert c.rows.shape[1] == 4  # L+1 = 2 padded to 4 (16-byte rows)


def test_node_range_rows_are_the_corpus_slice(mhw, oracle):
    """A start-node range yields exactly those walkers' rows, in corpus order
    (the per-GPU shard of a multi-GPU run)."""
    g = typed_random_graph(9, 120, 5.0)
    md = model_desc(O.DEEPWALK, g)
    dg, m = device_graph(g), walk_model(md)
    full = mhw.generate_walks(dg, m, mhw.WalkConfig(walks_per_node=3, walk_length=5, threads=8, seed=2))
    part = mhw.generate_walks(dg, m, mhw.WalkConfig(walks_per_node=3, walk_length=5, threads=8, seed=2,
                                                    node_begin=40, node_end=90))
    assert len(part) == 50 * 3
    assert np.array_equal(part.rows[:, 0], full.rows[40 * 3:90 * 3, 0])
    with pytest.raises(mhw.ValidationError, match="node range"):
        mhw.generate_walks(dg, m, mhw.WalkConfig(node_begin=5, node_end=500))


def test_asymmetric_adjacency_raises_like_update_state(mhw):
    """Flagged symmetric but missing back arcs: the walk fails with the
    reference's ValidationError message (models.cpp:131-133)."""
    # 0 -> 1, 1 -> 2, 2 -> 0 only (a directed triangle), flagged symmetric
    g = O.make_graph(3, [(0, 1, 1.0), (1, 2, 1.0), (2, 0, 1.0)], symmetric=True)
    dg = device_graph(g)
    assert not dg.info()["verified_symmetric"]
    O.assign_random_types(g, 2, O.XoRng(1))
    for kind in (O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK):
        for threads in (1, 8):
            with pytest.raises(mhw.ValidationError, match="asymmetric adjacency: no back edge"):
                mhw.generate_walks(device_graph(g), walk_model(model_desc(kind, g)),
                                   mhw.WalkConfig(walks_per_node=1, walk_length=5, threads=threads))


def test_dead_end_state_terminates_early(mhw, oracle):
    """metapath2vec on a node whose neighbours lack the required type: dead
    end (nullopt from mh_init) -> early termination, walk kept."""
    g = O.make_graph(3, [(0, 1, 1.0), (1, 0, 1.0), (1, 2, 1.0), (2, 1, 1.0)])
    g.ntype, g.n_ntypes = np.array([0, 1, 1], dtype=np.uint16), 2
    md = model_desc(O.METAPATH2VEC, g, metapath=(0, 1, 2 - 1, 0))
    for threads in (1, 8):
        c = mhw.generate_walks(device_graph(g), walk_model(md),
                               mhw.WalkConfig(walks_per_node=2, walk_length=10, threads=threads, seed=1))
        cfg = O.WalkCfg(K=2, L=10, seed=1)
        orow, olen, ost = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
        assert list(c.lengths) == list(olen)
        assert c.stats.early_terminations == ost["early_terminations"]


def test_one_chain_per_state_layout(mhw, oracle):
    """chain_replica_degree = 0xFFFFFFFF is SamplerManager's layout exactly."""
    rng = O.XoRng(21)
    g = O.preferential_attachment(200, 3, rng)
    md = model_desc(O.DEEPWALK, g)
    cfg = O.WalkCfg(K=4, L=20, seed=3)  # replica_degree default: none
    orow, olen, ost = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg))
    assert corpus_equal(orow, olen, c.rows, c.lengths)
    assert c.stats.slot_inits <= g.n


def _stats_dict(st):
    return dict(walks=st.walks, early_terminations=st.early_terminations, skipped_starts=st.skipped_starts,
                steps=st.steps, steps_per_sec=st.steps_per_sec, init_seconds=st.init_seconds,
                walk_seconds=st.walk_seconds)


@pytest.mark.parametrize("L", [1, 7, 80])
def test_device_corpus_text_equals_write_corpus(mhw, ref, tmp_path, L):
    """Text formatted on the GPU (mhw_generate_walks_to_file) and its stats
    sidecar == the REFERENCE's write_corpus (oracle/_ref, engine.cpp:236-259)
    of the same corpus and stats (deterministic schedule, so both runs
    agree), byte for byte."""
    import ctypes as C
    from paper_2010_04895_b200 import _lib as L_
    rng = O.XoRng(8)
    g = O.random_graph(2000, 4.0, True, rng, ensure_connected=False)   # isolated nodes too
    md = model_desc(O.DEEPWALK, g)
    cfgw = walk_config(O.WalkCfg(K=3, L=L, seed=4))
    dg, m = device_graph(g), walk_model(md)
    corpus = mhw.generate_walks(dg, m, cfgw)
    want = str(tmp_path / "want.txt")
    mhw.write_corpus(corpus, want)
    got = str(tmp_path / "got.txt")
    d, keep = m._desc()
    st = L_.WalkStatsC()
    assert L_.lib().mhw_generate_walks_to_file(dg.handle, C.byref(d), C.byref(cfgw._c()), got.encode(), C.byref(st)) == 0
    assert open(got, "rb").read() == open(want, "rb").read()
    assert st.steps == corpus.stats.steps
    refp = str(tmp_path / "ref.txt")
    ref.write_corpus(refp, corpus.rows, corpus.lengths, _stats_dict(st))
    for suffix in ("", ".stats.jsonl"):
        assert open(got + suffix, "rb").read() == open(refp + suffix, "rb").read(), suffix


def test_walks_write_matches_write_corpus_format(mhw, ref, tmp_path):
    """mhw_walks_write (C, host) == write_corpus's format (engine.cpp:236-247)."""
    import ctypes as C
    from paper_2010_04895_b200 import _lib as L
    g = typed_random_graph(4, 40, 3.0)
    md = model_desc(O.NODE2VEC, g)
    d, keep = walk_model(md)._desc()
    c = walk_config(O.WalkCfg(K=2, L=7, seed=5))._c()
    h = C.c_void_p()
    lib = L.lib()
    assert lib.mhw_generate_walks(device_graph(g).handle, C.byref(d), C.byref(c), C.byref(h)) == 0
    p = str(tmp_path / "c.txt")
    assert lib.mhw_walks_write(h, p.encode()) == 0
    rows = lib.mhw_walks_count(h)
    stride = lib.mhw_walks_stride(h)
    nodes = np.ctypeslib.as_array(C.cast(lib.mhw_walks_nodes(h), C.POINTER(C.c_uint32)), shape=(rows * stride,))
    lens = np.ctypeslib.as_array(C.cast(lib.mhw_walks_lengths(h), C.POINTER(C.c_uint32)), shape=(rows,))
    want = "".join(" ".join(str(int(x)) for x in nodes[r * stride:r * stride + lens[r]]) + "\n" for r in range(rows))
    st = L.WalkStatsC()
    assert lib.mhw_walks_stats(h, C.byref(st)) == 0
    rows_np = np.array(nodes).reshape(rows, stride)
    lens_np = np.array(lens)
    lib.mhw_walks_free(h)
    assert open(p).read() == want
    # the reference's own write_corpus of the same corpus and stats
    refp = str(tmp_path / "ref.txt")
    ref.write_corpus(refp, rows_np, lens_np, _stats_dict(st))
    for suffix in ("", ".stats.jsonl"):
        assert open(p + suffix, "rb").read() == open(refp + suffix, "rb").read(), suffix


def test_mega_hub_star(mhw):
    """A hub of degree 150,000 (past the 65,536-replica cap of the automatic
    deepwalk layout, with a 4,688-bucket hash set for the alpha test): walks
    stay valid, full length, and return to the hub every other step."""
    n = 150_001
    leaves = np.arange(1, n, dtype=np.int64)
    off = np.concatenate([[0, n - 1], n - 1 + np.arange(1, n)]).astype(np.int64)
    nbr = np.concatenate([leaves, np.zeros(n - 1, dtype=np.int64)]).astype(np.int32)
    w = (1.0 + (np.arange(2 * (n - 1)) % 7)).astype(np.float32)
    g = mhw.Graph.from_csr(off, nbr, weights=w, symmetric=True)
    for kind in (mhw.ModelKind.deepwalk, mhw.ModelKind.node2vec):
        m = mhw.WalkModel(kind=kind, p=0.5, q=2.0)
        c = mhw.generate_walks(g, m, mhw.WalkConfig(walks_per_node=2, walk_length=12, threads=8, seed=3))
        assert len(c) == 2 * n and (c.lengths == 13).all()
        rows = c.rows[:, :13].astype(np.int64)
        hub_pos = rows[:, 0] == 0
        # from the hub every step leaves it; from a leaf every step returns
        assert (rows[hub_pos][:, 1::2] != 0).all() and (rows[hub_pos][:, 2::2] == 0).all()
        assert (rows[~hub_pos][:, 1::2] == 0).all() and (rows[~hub_pos][:, 2::2] != 0).all()


def test_walk_rows_matches_corpus(mhw):
    """mhw_walk_rows sizes the caller's buffers without building a session:
    valid starts (metapath2vec: type == metapath[0]) in the node range x K."""
    import ctypes as C

    from paper_2010_04895_b200 import _lib as L
    rng = O.XoRng(44)
    g = O.random_graph(90, 4.0, True, rng, ensure_connected=False)
    O.assign_random_types(g, 2, rng)
    dg = device_graph(g)
    for kind in (O.DEEPWALK, O.METAPATH2VEC, O.NODE2VEC):
        m = walk_model(model_desc(kind, g))
        for b, e in ((0, 0), (10, 70)):
            cfg = mhw.WalkConfig(walks_per_node=3, walk_length=9, threads=8, seed=1, node_begin=b, node_end=e)
            d, keep = m._desc()
            c = cfg._c()
            rows, stride = C.c_uint64(), C.c_uint32()
            assert L.lib().mhw_walk_rows(dg.handle, C.byref(d), C.byref(c), C.byref(rows), C.byref(stride)) == 0
            corpus = mhw.generate_walks(dg, m, cfg)
            assert rows.value == len(corpus) and stride.value == 12


def test_manifest_of_a_run_equals_reference(mhw, ref, tmp_path):
    """cmd_walk's manifest for a device run: graph size and graph_checksum
    (computed from the device CSR) and T_i / T_w from the run's stats, in the
    reference's nlohmann dump(2) bytes."""
    rng = O.XoRng(31)
    g = O.random_graph(300, 5.0, True, rng)
    md = model_desc(O.NODE2VEC, g, p=0.5, q=2.0)
    cfg = O.WalkCfg(K=2, L=10, seed=9, init_kind=O.INIT_BURN_IN, burn_in_steps=7)
    dg, m, wc = device_graph(g), walk_model(md), walk_config(O.WalkCfg(K=2, L=10, seed=9, init_kind=O.INIT_BURN_IN,
                                                                       burn_in_steps=7), threads=8)
    c = mhw.generate_walks(dg, m, wc)
    out = str(tmp_path / "walks.txt")
    mhw.write_manifest(dg, m, wc, c.stats, out, input="g.txt", weighted=True, symmetrize=True)
    w = dg.download()["weights"].astype(np.float64)  # the device CSR's fp32 weights, widened
    want = ref.manifest(input="g.txt", weighted=1, symmetrize=1, model="node2vec", p=0.5, q=2.0,
                        walks_per_node=2, walk_length=10, sampler="mh", init="burn_in", burn_in_steps=7,
                        hw_sample_size=wc.init.hw_sample_size, threads=8, seed=9, output=out, nodes=g.n, arcs=g.m,
                        checksum=O.Oracle().graph_checksum(g.offsets, g.nbr, w), T_i=c.stats.init_seconds,
                        T_w=c.stats.walk_seconds)
    assert open(out + ".manifest.json", "rb").read() == want
