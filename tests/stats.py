"""Distribution checks for M-H walk corpora.

Outputs of one M-H chain are autocorrelated, so a multinomial chi-square
over them is not valid (the reference's own tests use KL/L-inf
tolerances for that reason). The per-state outputs of the engine ARE the
trajectory of that state's chain (every visit is one transition of the
uniform-proposal M-H kernel P, samplers.hpp:18-27), so the Markov-chain CLT
applies: sqrt(N)(p_hat - pi) -> N(0, S) with
    S = diag(pi) Z + Z^T diag(pi) - diag(pi) - pi pi^T,
    Z = (I - P + 1 pi^T)^-1            (Kemeny-Snell fundamental matrix),
and N (p_hat - pi)^T S^+ (p_hat - pi) ~ chi2(d - 1). That is the
"chi-square test at p >= 0.01" of the north star, computed exactly.
"""
from __future__ import annotations

from collections import defaultdict

import numpy as np
from scipy import stats as st

from oracle import oracle as O


def mh_kernel(pi: np.ndarray, proposals: int | None = None) -> np.ndarray:
    """Exact uniform-proposal M-H kernel (tests/oracles.hpp:207-220) on the
    support pi; `proposals` = size of the proposal set (the full degree:
    zero-weight candidates are proposed too and always rejected,
    samplers.hpp:21)."""
    n = len(pi)
    m = proposals or n
    P = np.zeros((n, n))
    for i in range(n):
        with np.errstate(divide="ignore", invalid="ignore"):
            P[i] = np.minimum(1.0, np.where(pi[i] > 0, pi / pi[i], 1.0)) / m
        P[i, i] = 0.0
        P[i, i] = 1.0 - P[i].sum()
    return P


def markov_chi2(counts: np.ndarray, pi: np.ndarray) -> tuple[float, int, float]:
    """(statistic, dof, p-value) of the chain-CLT chi-square on the support."""
    sup = pi > 0
    pi_s = pi[sup] / pi[sup].sum()
    c = counts[sup].astype(np.float64)
    if counts[~sup].sum() > 0:
        return float("inf"), 0, 0.0  # zero-weight candidate emitted
    n = len(pi_s)
    if n < 2:
        return 0.0, 0, 1.0
    P = mh_kernel(pi_s, proposals=len(pi))
    Z = np.linalg.inv(np.eye(n) - P + np.outer(np.ones(n), pi_s))
    D = np.diag(pi_s)
    S = D @ Z + Z.T @ D - D - np.outer(pi_s, pi_s)
    N = c.sum()
    d = c / N - pi_s
    stat = float(N * d @ np.linalg.pinv(S, rcond=1e-10, hermitian=True) @ d)
    dof = n - 1
    return stat, dof, float(st.chi2.sf(stat, dof))


def transitions(rows, lens, kind, metapath=None):
    """state -> {next node: count}. States: deepwalk v; metapath2vec
    (v, position mod cycle); second order (prev, v) after the bootstrap step."""
    out = defaultdict(lambda: defaultdict(int))
    for r in range(len(lens)):
        w = rows[r, :lens[r]].tolist()
        a = 0
        for i in range(len(w) - 1):
            if kind == O.DEEPWALK:
                key = w[i]
            elif kind == O.METAPATH2VEC:
                # the chain is keyed by (v, required next type) (models.cpp:167, Q6)
                key = (w[i], int(metapath[_next(a, metapath)]))
                a = _next(a, metapath)
            else:
                if i == 0:
                    continue  # bootstrap step: static weights, no chain
                key = (w[i - 1], w[i])
            out[key][w[i + 1]] += 1
    return out


def _next(a, mp):
    """metapath_next (models.hpp:82-85)."""
    return a + 1 if a + 1 < len(mp) else (1 if mp[0] == mp[-1] and len(mp) > 1 else 0)


def _mp_index(i, mp):
    a = 0
    for _ in range(i):
        a = _next(a, mp)
    return a


def audit(g: O.HostGraph, oracle: O.Oracle, md: O.ModelDesc, rows, lens, min_visits=5000, max_states=40):
    """p-values of the chain chi-square for states visited >= min_visits."""
    tr = transitions(rows, lens, md.kind, md.metapath)
    pv = []
    for key, nxt in sorted(tr.items(), key=lambda kv: -sum(kv[1].values()))[:max_states]:
        visits = sum(nxt.values())
        if visits < min_visits:
            break
        if md.kind == O.DEEPWALK:
            v, aff = key, O.NO_AFFIX
        elif md.kind == O.METAPATH2VEC:
            v, req = key
            aff = next(a for a in range(len(md.metapath)) if md.metapath[_next(a, md.metapath)] == req)
        else:
            s, v = key
            aff = int(np.searchsorted(g.neighbors_of(v), s))
        pi = O.eval_target(g, oracle, md, v, aff)
        nb = g.neighbors_of(v)
        counts = np.zeros(len(nb))
        for u, cnt in nxt.items():
            counts[int(np.searchsorted(nb, u))] += cnt
        pv.append(markov_chi2(counts, pi)[2])
    return np.array(pv)


def gate(pvals: np.ndarray, alpha=0.01, family=1e-4):
    """Family check at false-alarm rate ~3 x `family` per call: no state
    below the Bonferroni floor family / n, Fisher's combined p >= family, and
    the count of per-state p < alpha (the north star's p >= 0.01 criterion)
    consistent with chance (binomial tail >= family). A suite makes ~20
    calls, so spurious failures stay below 1%; real biases (a 10%
    mis-weighted target, the lost-update CAS chain) score p < 1e-20."""
    if len(pvals) == 0:
        return False, "no audited states"
    n = len(pvals)
    fisher = st.combine_pvalues(np.maximum(pvals, 1e-300), method="fisher").pvalue
    low = int(np.sum(pvals < alpha))
    binom = st.binom.sf(low - 1, n, alpha) if low else 1.0
    ok = pvals.min() >= family / n and fisher >= family and binom >= family
    return ok, f"n={n} min={pvals.min():.2e} fisher={fisher:.2e} low={low} binom={binom:.2e}"
