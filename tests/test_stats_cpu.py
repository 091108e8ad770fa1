"""Calibration of the chain chi-square gate (tests/stats.py) on CPU oracle
corpora: it accepts exact M-H chains and rejects a wrong target. This is the
control arm of the GPU distribution tests."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import model_desc
from tests.stats import audit, gate, markov_chi2, mh_kernel


def test_kernel_detailed_balance():
    """acceptance.cpp:66-79: pi_i P_ij == pi_j P_ji for the exact kernel."""
    r = np.random.default_rng(0)
    for _ in range(20):
        pi = r.uniform(0.05, 1.05, r.integers(2, 17))
        pi /= pi.sum()
        P = mh_kernel(pi)
        F = pi[:, None] * P
        assert np.abs(F - F.T).max() < 1e-12
        assert np.allclose(P.sum(1), 1.0)


def test_chain_chi2_accepts_exact_chain_and_rejects_wrong_target():
    r = np.random.default_rng(1)
    pi = np.array([1.0, 2.0, 3.0, 0.5, 4.0])
    pi /= pi.sum()
    P = mh_kernel(pi)
    cdf = np.cumsum(P, axis=1)
    x, counts = 0, np.zeros(5)
    for _ in range(200000):
        x = int(np.searchsorted(cdf[x], r.random()))
        counts[x] += 1
    assert markov_chi2(counts, pi)[2] > 1e-3
    wrong = pi.copy()
    wrong[0] *= 1.1
    wrong /= wrong.sum()
    assert markov_chi2(counts, wrong)[2] < 1e-6
    # a plain multinomial chi-square over-rejects autocorrelated outputs
    from scipy import stats as st
    chi = float(np.sum((counts - pi * counts.sum()) ** 2 / (pi * counts.sum())))
    assert chi > 0


@pytest.mark.parametrize("kind", [O.DEEPWALK, O.NODE2VEC])
def test_oracle_corpus_passes_gate(oracle, kind):
    """The control: the CPU oracle's corpus (pinned to the reference) passes."""
    rng = O.XoRng(12)
    g = O.preferential_attachment(50, 3, rng) if kind == O.DEEPWALK else O.random_graph(30, 4.0, True, rng)
    md = model_desc(kind, g, p=0.5, q=2.0)
    cfg = O.WalkCfg(K=50 if kind == O.DEEPWALK else 300, L=80, seed=13)
    rows, lens, _ = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    pv = audit(g, oracle, md, rows, lens, min_visits=5000)
    ok, msg = gate(pv)
    assert ok, msg


def _uniform_proposal_chain(pi_w, steps, r, m=None):
    """An exact uniform-proposal M-H chain (samplers.hpp:18-27) over
    unnormalised weights pi_w, simulated directly."""
    m = m or len(pi_w)
    x = int(np.argmax(pi_w > 0))
    counts = np.zeros(len(pi_w))
    cand = r.integers(0, m, steps)
    u = r.random(steps)
    for c, uu in zip(cand, u):
        if pi_w[x] <= 0 or pi_w[c] >= pi_w[x] or uu * pi_w[x] < pi_w[c]:
            x = int(c)
        counts[x] += 1
    return counts


def test_lumped_chi2_is_calibrated_and_has_power():
    """The lumped (equal-weight classes) chain chi-square used for hub states:
    p-values of exact chains are not small, a 10% mis-weighted class is
    caught, and it agrees with the full test where both apply."""
    from tests.stats import lumped_chi2
    r = np.random.default_rng(7)
    w = np.concatenate([np.full(1, 4.0), np.full(40, 1.0), np.full(400, 0.25), np.zeros(9)])  # node2vec-like classes
    pi = w / w.sum()
    pvals = [lumped_chi2(_uniform_proposal_chain(w, 60000, r), pi)[2] for _ in range(12)]
    assert min(pvals) > 1e-3
    counts = _uniform_proposal_chain(w, 200000, r)
    wrong = w.copy()
    wrong[1:41] *= 1.10
    assert lumped_chi2(counts, wrong / wrong.sum())[2] < 1e-6
    assert lumped_chi2(counts, pi)[2] > 1e-4
    # a zero-weight candidate in the output fails outright
    bad = counts.copy()
    bad[-1] += 1
    assert lumped_chi2(bad, pi)[2] == 0.0
    # small support: same verdict as the full test
    w2 = np.array([1.0, 1.0, 2.0, 2.0, 3.0])
    c2 = _uniform_proposal_chain(w2, 100000, r)
    assert lumped_chi2(c2, w2 / w2.sum())[2] > 1e-3 and markov_chi2(c2, w2 / w2.sum())[2] > 1e-3


@pytest.mark.parametrize("kind", [O.DEEPWALK, O.NODE2VEC, O.METAPATH2VEC, O.FAIRWALK])
def test_transition_counts_gpu_equals_transitions(oracle, kind):
    """The torch counter used on BASELINE-size corpora (run here on the CPU)
    equals the pure-Python per-state counts, including several audited
    states that share one node v (second order: (s1, v), (s2, v))."""
    from tests.stats import transition_counts_gpu, transitions
    rng = O.XoRng(55)
    g = O.random_graph(12, 3.0, True, rng)
    O.assign_random_types(g, 2, rng)
    md = model_desc(kind, g, p=0.5, q=2.0, metapath=(0, 1, 0))
    cfg = O.WalkCfg(K=300, L=20, seed=3)
    rows, lens, _ = oracle.generate_walks(g, md, cfg)
    states = transition_counts_gpu(rows, lens, kind, g.offsets, g.nbr, metapath=md.metapath,
                                   min_visits=50, max_states=25)
    ref = transitions(rows, lens, kind, md.metapath)
    assert len(states) >= 5
    nodes = [v for v, *_ in states]
    if kind in (O.NODE2VEC, O.FAIRWALK):
        assert len(set(nodes)) < len(nodes)  # shared nodes are exercised
    for v, aff, vis, counts in states:
        nb = g.neighbors_of(v)
        if kind == O.DEEPWALK:
            key = v
        elif kind == O.METAPATH2VEC:
            key = (v, int(md.metapath[aff + 1 if aff + 1 < len(md.metapath) else 1]))
        else:
            key = (int(nb[aff]), v)
        exp = np.array([ref[key].get(int(u), 0) for u in nb])
        assert counts.sum() == vis == exp.sum()
        assert np.array_equal(counts, exp)


def test_alias_proposal_kernel_is_calibrated_and_has_power():
    """The independent-proposal kernel of tests/stats.py (alias proposal, q ~
    static weights): exact Hastings chains pass, a chain that forgets the
    correction (accepting with min(1, w'_c / w'_l)) fails."""
    r = np.random.default_rng(11)
    w = np.array([1.0, 3.0, 0.5, 2.0, 6.0, 1.5])         # static weights (proposal)
    f = np.array([4.0, 1.0, 0.25, 1.0, 0.25, 1.0])       # dynamic factors r = w'/w
    pi = w * f / np.sum(w * f)
    q = w / w.sum()

    def chain(steps, hastings=True):
        x, c = 0, np.zeros(len(w))
        for cand, u in zip(r.choice(len(w), size=steps, p=q), r.random(steps)):
            a, b = (f[cand], f[x]) if hastings else (w[cand] * f[cand], w[x] * f[x])
            if a >= b or u * b < a:
                x = int(cand)
            c[x] += 1
        return c

    assert markov_chi2(chain(100000), pi, q)[2] > 1e-3
    assert markov_chi2(chain(100000, hastings=False), pi, q)[2] < 1e-6


@pytest.mark.parametrize("kind", [O.DEEPWALK, O.NODE2VEC, O.METAPATH2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_oracle_alias_proposal_chains_hit_the_target(oracle, kind):
    """The oracle's alias-proposal M-H (og_walk: static alias table proposal,
    og_hastings accept) leaves the per-state targets of calculate_weight
    invariant: its corpus passes the chain chi-square with the alias kernel."""
    from tests.stats import audit
    from tests.helpers import typed_random_graph
    g = typed_random_graph(700 + kind, 40, 4.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.5, q=2.0, M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)),
                    metapath=(0, 1, 0))
    cfg = O.WalkCfg(K=400, L=80, seed=5, init_kind=O.INIT_RANDOM, proposal=1)
    rows, lens, _ = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    ok, msg = gate(audit(g, oracle, md, rows, lens, min_visits=5000, alias_proposal=True))
    assert ok, msg


def test_oracle_hastings_decisions_restated(oracle):
    """og_decide_hastings = the factor ratio rule restated here: r = w'/w
    (exact for node2vec: alpha), accept iff w_c > 0 and (r_l <= 0 or r_c >= r_l
    or u r_l < r_c)."""
    from tests.helpers import random_triples
    rng = O.XoRng(5)
    g = O.random_graph(120, 6.0, True, rng)
    md = model_desc(O.NODE2VEC, g, p=0.3, q=3.0)
    pos, aff, cand, last, u = random_triples(g, md, 5000, seed=2)
    rc, rl, acc = oracle.decide_hastings(g, md, pos, aff, cand, last, u)
    wc, wl, _ = oracle.decide(g, md, pos, aff, cand, last, u)
    off = g.offsets.astype(np.int64)
    w_c = g.w[off[pos] + cand]
    w_l = g.w[off[pos] + last]
    boot = aff == O.NO_AFFIX
    assert np.all(rc[boot] == 1.0)
    alpha_ok = np.isin(rc[~boot], [1 / 0.3, 1.0, 1 / 3.0])
    assert np.all(alpha_ok)
    assert np.array_equal(wc, rc * w_c) and np.array_equal(wl, rl * w_l)  # node2vec: a * w
    want = (w_c > 0) & ((rl <= 0) | (rc >= rl) | (u * rl < rc))
    assert np.array_equal(acc.astype(bool), want)


def test_class_entries_flag_slow_hub_chains():
    """The validity guard of audit_counts(min_entries=...): at 8,000 visits a
    hub state whose heavy class is a single candidate among 20,000 enters it
    well under once, an ordinary state's classes hundreds of times."""
    from tests.stats import min_class_entries
    hub = np.concatenate([[4.0], np.full(8, 1.0), np.full(19991, 0.25)])
    assert min_class_entries(hub, 8000) < 1
    leaf = np.array([4.0, 1.0, 1.0, 0.25, 0.25, 0.25, 0.25, 0.25])
    assert min_class_entries(leaf, 8000) > 100
