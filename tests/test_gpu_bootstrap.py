"""Weighted bootstrap (direct_sample, samplers.cpp:133-146, first step of a
second-order walk, engine.cpp:81-83) on hub slices: the device resumes the
reference's sequential scan at the block located through exact block prefix
sums (k_wblk), or scans the whole slice where exactness is not guaranteed.
Either way the first step of every walk equals the oracle's sequential scan
byte for byte (deterministic schedule vs the oracle's Philox step-major mode)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import corpus_equal, device_graph, model_desc, walk_config, walk_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def hub_graph(seed, hubs, hub_deg, leaves, weight_fn) -> O.HostGraph:
    """`hubs` hubs joined to `hub_deg` random leaves each, plus a ring over the
    leaves; weights per undirected edge from weight_fn(rng) (fp32 values)."""
    rng = np.random.default_rng(seed)
    n = hubs + leaves
    pairs = set()
    for h in range(hubs):
        for x in rng.choice(leaves, hub_deg, replace=False):
            pairs.add((h, hubs + int(x)))
    for i in range(leaves):
        a, b = hubs + i, hubs + (i + 1) % leaves
        pairs.add((min(a, b), max(a, b)))
    edges = []
    for a, b in sorted(pairs):
        w = float(np.float32(weight_fn(rng)))
        edges += [(a, b, w), (b, a, w)]
    return O.make_graph(n, edges)


WEIGHTS = {
    "uniform": lambda r: r.uniform(1.0, 10.0),
    "dyadic": lambda r: 2.0 ** int(r.integers(-3, 4)),       # ties with block prefixes
    "wide": lambda r: 10.0 ** r.uniform(-30, 30),            # no exactness guarantee: full scan
    "zeros": lambda r: 0.0 if r.uniform() < 0.3 else r.uniform(0.5, 2.0),
}


@pytest.mark.parametrize("wname", sorted(WEIGHTS))
@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_hub_bootstrap_equals_sequential_scan(mhw, oracle, kind, wname):
    g = hub_graph(11 + kind, hubs=3, hub_deg=1500, leaves=2000, weight_fn=WEIGHTS[wname])
    O.assign_random_types(g, 2, O.XoRng(5))
    md = model_desc(kind, g, p=0.5, q=2.0)
    cfg = O.WalkCfg(K=40, L=3, seed=91, init_kind=O.INIT_RANDOM)
    orow, olen, _ = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=1))
    assert corpus_equal(orow, olen, c.rows, c.lengths)
    # the hubs' walkers took their first step through the block search
    hub_rows = np.nonzero(orow[:, 0] < 3)[0]
    assert len(hub_rows) == 3 * cfg.K and (olen[hub_rows] > 1).all()


def test_throughput_bootstrap_first_steps_equal_deterministic(mhw, oracle):
    """The throughput schedule draws the bootstrap from the same (walker, step 0)
    Philox block, so the first step of every walk is identical across schedules."""
    g = hub_graph(3, hubs=4, hub_deg=3000, leaves=4000, weight_fn=WEIGHTS["uniform"])
    md = model_desc(O.NODE2VEC, g, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=64, L=2, seed=5, init_kind=O.INIT_RANDOM)
    dg = device_graph(g)
    det = mhw.generate_walks(dg, walk_model(md), walk_config(cfg, threads=1))
    thr = mhw.generate_walks(dg, walk_model(md), walk_config(cfg, threads=8))
    assert np.array_equal(det.rows[:, :2], thr.rows[:, :2])
