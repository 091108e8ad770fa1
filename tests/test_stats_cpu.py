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
