"""og_walk_isolated -- a walker alone with a fresh SamplerManager (the checker
of the single-walker k_walk pin, tests/test_gpu_kwalk_pin.py) -- against the
oracle's own walker-major run: the first walker of a walker-major run
(engine.cpp:178-205, threads = 1) also starts from an empty manager, so the two
must agree byte for byte, for every model, init strategy and chain layout."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import INITS, KINDS, model_desc, typed_random_graph


@pytest.mark.parametrize("init", INITS)
@pytest.mark.parametrize("kind", KINDS)
def test_isolated_walker_equals_first_walker_of_a_run(oracle, kind, init):
    g = typed_random_graph(60 + kind, 50, 6.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.3, q=3.0, metapath=(0, 1, 0),
                    M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)))
    for rep in (0xFFFFFFFF, 0, 1):  # one chain per state, automatic replicas, replicas everywhere
        cfg = O.WalkCfg(K=1, L=30, seed=5 + kind, init_kind=init, burn_in_steps=4, hw_sample_size=4,
                        replica_degree=rep)
        rows, lens, st = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_WALKER)
        v0 = int(rows[0, 0])  # the first valid start
        irows, ilens, ist = oracle.walk_isolated(g, md, cfg, [v0])
        assert ilens[0] == lens[0]
        assert np.array_equal(irows[0, :ilens[0]], rows[0, :lens[0]])


def test_isolated_walkers_are_independent_of_each_other(oracle):
    """Several starts in one call = the same starts one call each."""
    g = typed_random_graph(77, 60, 5.0, weighted=True, types=2)
    md = model_desc(O.NODE2VEC, g, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=2, L=25, seed=3, init_kind=O.INIT_BURN_IN, burn_in_steps=5)
    starts = [1, 7, 30, 59]
    rows, lens, st = oracle.walk_isolated(g, md, cfg, starts)
    assert len(lens) == 8 and st["walks"] == 8
    for j, v in enumerate(starts):
        r1, l1, _ = oracle.walk_isolated(g, md, cfg, [v])
        for k in range(2):
            assert np.array_equal(rows[2 * j + k, :lens[2 * j + k]], r1[k, :l1[k]])
