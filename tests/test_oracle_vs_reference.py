"""Live comparison of the C restatement against the compiled reference
(oracle/_ref) over randomized graphs; skipped where the reference tree and
library are absent (e.g. on the GPU box)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import INITS, KINDS, model_desc, random_triples


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("kind", KINDS)
def test_corpus_byte_identical(oracle, ref, seed, kind):
    rng = O.XoRng(1000 + seed)
    g = O.random_graph(40 + 30 * seed, 4.0 + seed, seed != 2, rng, ensure_connected=seed != 3)
    O.assign_random_types(g, 2 + seed % 2, rng)
    for init in INITS:
        md = model_desc(kind, g, p=0.25 + 0.3 * seed, q=4.0 / seed,
                        metapath=(0, 1, 0) if seed % 2 else (0, 1))
        if kind == O.EDGE2VEC:
            md.type_matrix = np.random.default_rng(seed).uniform(0.1, 1.1, md.type_matrix.shape)
        cfg = O.WalkCfg(K=3, L=15, seed=seed * 7, init_kind=init, burn_in_steps=5, hw_sample_size=3)
        rows, lens, st = oracle.generate_walks(g, md, cfg)
        rr, rl, rs = ref.graph(g).model(md).generate_walks(cfg, threads=1, n_nodes=g.n)
        assert np.array_equal(lens, rl)
        for i in range(len(lens)):
            assert np.array_equal(rows[i, :lens[i]], rr[i, :rl[i]])
        assert st["steps"] == rs["steps"] and st["early_terminations"] == rs["early_terminations"]


@pytest.mark.parametrize("sampler", [O.SAMPLER_ALIAS, O.SAMPLER_DIRECT, O.SAMPLER_REJECTION])
@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("kind", KINDS)
def test_baseline_sampler_corpus_byte_identical(oracle, ref, seed, kind, sampler):
    """The exact baselines of next_edge (engine.cpp:88-116): alias tables per
    state slot, direct inverse-CDF, rejection under a static alias proposal
    with the rejection_bound envelope -- same corpus as generate_walks."""
    rng = O.XoRng(2000 + seed)
    g = O.random_graph(50 + 20 * seed, 4.0 + seed, seed != 2, rng, ensure_connected=seed != 1)
    O.assign_random_types(g, 2 + seed % 2, rng)
    md = model_desc(kind, g, p=0.5 + 0.2 * seed, q=2.0 / seed, metapath=(0, 1, 0) if seed % 2 else (0, 1))
    if kind == O.EDGE2VEC:
        md.type_matrix = np.random.default_rng(seed).uniform(0.1, 1.1, md.type_matrix.shape)
    cfg = O.WalkCfg(K=3, L=15, seed=seed * 11, sampler=sampler)
    rows, lens, st = oracle.generate_walks(g, md, cfg)
    rr, rl, rs = ref.graph(g).model(md).generate_walks(cfg, threads=1, n_nodes=g.n)
    assert np.array_equal(lens, rl)
    for i in range(len(lens)):
        assert np.array_equal(rows[i, :lens[i]], rr[i, :rl[i]])
    assert st["steps"] == rs["steps"] and st["early_terminations"] == rs["early_terminations"]


@pytest.mark.parametrize("kind", KINDS)
def test_decisions_bit_exact(oracle, ref, kind):
    rng = O.XoRng(77 + kind)
    g = O.random_graph(150, 7.0, True, rng)
    O.assign_random_types(g, 3, rng)
    md = model_desc(kind, g, p=0.3, q=3.3, metapath=(0, 2, 1, 0),
                    M=np.random.default_rng(kind).uniform(0.5, 2.0, (9, 9)))
    pos, aff, cand, last, u = random_triples(g, md, 20000, seed=kind)
    a = oracle.decide(g, md, pos, aff, cand, last, u)
    b = ref.graph(g).model(md).decide(pos, aff, cand, last, u)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_model_bind_errors_match(oracle, ref):
    """bind validation (models.cpp:29-74): asymmetric graph, missing types,
    bad metapath, matrix dimensions -> ValidationError (status 2) on both."""
    g = O.make_graph(2, [(0, 1, 1.0)], symmetric=False)
    for md in (O.ModelDesc(O.NODE2VEC), O.ModelDesc(O.METAPATH2VEC, metapath=[0, 1])):
        with pytest.raises(O.OracleError) as e1:
            oracle.bind(g, md)
        with pytest.raises(O.OracleError) as e2:
            ref.graph(g).model(md)
        assert e1.value.code == e2.value.code == 2


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("threads", [1, 3])
def test_sliced_full_run_equals_generate_walks(ref, kind, threads):
    """bench.py --impl reference: one full run in time slices over one shared
    SamplerManager (ref_run_slice) walks every walker exactly once with the
    generate_walks partition, so its counts equal generate_walks' (and with one
    thread, where the run is deterministic, every slot sees the same chain)."""
    rng = O.XoRng(3000 + kind)
    g = O.random_graph(90, 5.0, True, rng)
    O.assign_random_types(g, 2, rng)
    md = model_desc(kind, g, p=0.5, q=2.0, metapath=(0, 1, 0))
    cfg = O.WalkCfg(K=3, L=12, seed=5, init_kind=O.INIT_BURN_IN, burn_in_steps=4)
    rm = ref.graph(g).model(md)
    _, _, rs = rm.generate_walks(cfg, threads=threads, n_nodes=g.n, with_rows=False)
    run = rm.full_run(cfg, threads)
    tot = dict(walks=0, early_terminations=0, skipped_starts=0, steps=0)
    for i in range(5):
        st = run.slice(i, 5)
        for k in tot:
            tot[k] += st[k]
    assert tot["walks"] == rs["walks"] and tot["skipped_starts"] == rs["skipped_starts"]
    if threads == 1:
        assert tot["steps"] == rs["steps"] and tot["early_terminations"] == rs["early_terminations"]
