"""The exact baseline samplers (alias / direct / rejection, engine.cpp:88-116)
in the oracle's Philox layout: draws are keyed by (walker, step[, trial]) and
the per-state tables are deterministic, so the corpus cannot depend on the
walker schedule -- the property the GPU kernel (exact.cu) relies on."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import KINDS, model_desc

SAMPLERS = [O.SAMPLER_ALIAS, O.SAMPLER_DIRECT, O.SAMPLER_REJECTION]


@pytest.mark.parametrize("sampler", SAMPLERS)
@pytest.mark.parametrize("kind", KINDS)
def test_philox_corpus_is_schedule_free(oracle, kind, sampler):
    rng = O.XoRng(40 + kind)
    g = O.random_graph(70, 5.0, True, rng)
    O.assign_random_types(g, 3, rng)
    md = model_desc(kind, g, p=0.4, q=2.5, metapath=(0, 1, 2, 1, 0),
                    M=np.random.default_rng(kind).uniform(0.2, 1.5, (9, 9)))
    cfg = O.WalkCfg(K=3, L=20, seed=9, sampler=sampler)
    a = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_WALKER)
    b = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    assert np.array_equal(a[1], b[1])
    for i in range(len(a[1])):
        assert np.array_equal(a[0][i, :a[1][i]], b[0][i, :b[1][i]])
    assert a[2]["steps"] == b[2]["steps"] and a[2]["trials"] == b[2]["trials"]


@pytest.mark.parametrize("sampler", SAMPLERS)
def test_exact_samplers_hit_the_exact_target(oracle, sampler):
    """Pooled next-node frequencies from one state match the normalised w'
    (tools/mhwalk.cpp:208-220) -- exact sampling, no chain burn-in."""
    und = [(0, 1, 1.0), (0, 2, 3.0), (0, 3, 6.0), (1, 2, 2.0)]
    g = O.make_graph(4, und + [(b, a, w) for a, b, w in und])
    md = model_desc(O.NODE2VEC, g, p=0.5, q=2.0)
    # every walk starts at node 0 (bootstrap) then samples from states (prev, cur)
    cfg = O.WalkCfg(K=20000, L=2, seed=3, sampler=sampler)
    rows, lens, _ = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    sel = (rows[:, 0] == 0) & (rows[:, 1] == 2) & (lens == 3)
    nxt = rows[sel, 2]
    # state (prev 0, cur 2): N(2) = {0, 1} -> w' = {w(2,0)/p, w(2,1)*1 (1 adj 0)}
    target = np.array([3.0 / 0.5, 2.0 * 1.0])
    target /= target.sum()
    freq = np.array([(nxt == 0).mean(), (nxt == 1).mean()])
    assert sel.sum() > 3000
    assert np.allclose(freq, target, atol=0.03)


def low_acceptance_graph():
    """Triangle whose every arc has edge type 0 while edge2vec's M[0][0] is
    1e-6 of the envelope: a rejection step needs ~10^6 trials, far past the
    65536 trials one sub-counter epoch holds (the trial field of the
    sub-counter used to wrap and replay earlier trials forever)."""
    g = O.triangle()
    g.ntype, g.n_ntypes = np.zeros(3, dtype=np.uint16), 1
    g.etype, g.n_etypes = np.zeros(6, dtype=np.uint16), 2
    md = model_desc(O.EDGE2VEC, g, p=1.0, q=1.0, M=np.array([[1e-6, 1.0], [1.0, 1.0]]))
    return g, md


def test_rejection_streams_do_not_wrap(oracle):
    g, md = low_acceptance_graph()
    cfg = O.WalkCfg(K=1, L=3, seed=11, sampler=O.SAMPLER_REJECTION)
    rows, lens, st = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    assert st["steps"] == 9 and st["trials"] > 6 * 65536
    # every emitted node is a neighbour: the walk terminated normally
    for r in range(3):
        w = rows[r, :lens[r]]
        assert all(int(b) in g.neighbors_of(int(a)) for a, b in zip(w[:-1], w[1:]))
