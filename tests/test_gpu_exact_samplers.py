"""GPU exact baseline samplers (exact.cu) against the oracle's Philox layout:
byte-identical corpora and stats for every model x {alias, direct,
rejection}, on weighted / unweighted graphs with dead ends, plus the alias
memory guard. The oracle itself is pinned to the reference's generate_walks
for these samplers in test_oracle_vs_reference.py."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import KINDS, corpus_equal, device_graph, model_desc, walk_config, walk_model

pytestmark = pytest.mark.gpu
SAMPLERS = [O.SAMPLER_ALIAS, O.SAMPLER_DIRECT, O.SAMPLER_REJECTION]


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def _graph(seed, n, deg, weighted, connected=True):
    rng = O.XoRng(seed)
    g = O.random_graph(n, deg, weighted, rng, ensure_connected=connected)
    O.assign_random_types(g, 3, rng)
    return g


@pytest.mark.parametrize("weighted", [True, False])
@pytest.mark.parametrize("sampler", SAMPLERS)
@pytest.mark.parametrize("kind", KINDS)
def test_exact_sampler_corpus_equals_oracle(mhw, oracle, kind, sampler, weighted):
    g = _graph(300 + kind, 90, 6.0, weighted, connected=weighted)
    md = model_desc(kind, g, p=0.25, q=4.0, metapath=(0, 1, 2, 1, 0),
                    M=np.random.default_rng(kind).uniform(0.0, 1.5, (9, 9)))
    cfg = O.WalkCfg(K=4, L=25, seed=17, sampler=sampler)
    orow, olen, ost = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    c = mhw.generate_walks(device_graph(g, weighted=weighted), walk_model(md), walk_config(cfg, threads=8))
    assert corpus_equal(orow, olen, c.rows, c.lengths)
    s = c.stats
    assert (s.walks, s.early_terminations, s.skipped_starts, s.steps) == (
        ost["walks"], ost["early_terminations"], ost["skipped_starts"], ost["steps"])
    if sampler == O.SAMPLER_REJECTION:
        assert s.rejection_trials == ost["trials"]


@pytest.mark.parametrize("sampler", SAMPLERS)
def test_exact_sampler_hub_degrees(mhw, oracle, sampler):
    """Degrees well past one warp round (and past the 256-entry weight cache):
    the shuffle-replayed sequential sums must still match bit for bit."""
    r = np.random.default_rng(5)
    n = 600
    und = {(0, v) for v in range(1, 420)}  # a hub of degree 419
    while len(und) < 2400:
        a, b = sorted(int(x) for x in r.integers(1, n, 2))
        if a != b:
            und.add((a, b))
    w = {e: float(np.float32(0.5 + 3 * r.random())) for e in und}
    g = O.make_graph(n, [(a, b, w[(a, b)]) for a, b in und] + [(b, a, w[(a, b)]) for a, b in und])
    for kind in (O.NODE2VEC, O.DEEPWALK):
        md = model_desc(kind, g, p=0.5, q=2.0)
        cfg = O.WalkCfg(K=3, L=30, seed=4, sampler=sampler)
        orow, olen, _ = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
        c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=8))
        assert corpus_equal(orow, olen, c.rows, c.lengths)
    assert int(np.diff(g.offsets).max()) > 256


def test_alias_memory_guard(mhw):
    """Per-state alias tables for a second-order model need 12 B x sum deg^2:
    refused with a validation error instead of running out of memory."""
    g = mhw.Graph.rmat(20, 16, seed=1)
    m = mhw.WalkModel(kind=mhw.ModelKind.node2vec, p=0.25, q=4.0)
    cfg = mhw.WalkConfig(walks_per_node=1, walk_length=4, threads=8, sampler_kind=mhw.SamplerKind.alias)
    with pytest.raises(mhw.ValidationError, match="alias tables need"):
        mhw.generate_walks(g, m, cfg)


def test_rejection_past_one_trial_epoch_equals_oracle(mhw, oracle):
    """~10^6 rejection trials per step (acceptance 1e-6): the GPU's warp rounds
    cross many 65536-trial key epochs and still equal the oracle's draws."""
    from tests.test_exact_samplers_cpu import low_acceptance_graph
    g, md = low_acceptance_graph()
    cfg = O.WalkCfg(K=1, L=3, seed=11, sampler=O.SAMPLER_REJECTION)
    orow, olen, ost = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=8))
    assert corpus_equal(orow, olen, c.rows, c.lengths)
    assert c.stats.rejection_trials == ost["trials"] > 6 * 65536
