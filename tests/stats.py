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


def mh_kernel(pi: np.ndarray, proposals: int | None = None, q: np.ndarray | None = None) -> np.ndarray:
    """Exact M-H kernel on the support pi. Uniform proposal (tests/oracles.hpp:
    207-220): `proposals` = size of the proposal set (the full degree:
    zero-weight candidates are proposed too and always rejected,
    samplers.hpp:21). Independent proposal q (the alias proposal, q ~ static
    weights; q over the support, summing to <= 1 when some proposals fall
    outside it and are rejected): P_ij = q_j min(1, (pi_j / q_j) / (pi_i / q_i))."""
    n = len(pi)
    P = np.zeros((n, n))
    for i in range(n):
        with np.errstate(divide="ignore", invalid="ignore"):
            if q is None:
                P[i] = np.minimum(1.0, np.where(pi[i] > 0, pi / pi[i], 1.0)) / (proposals or n)
            else:
                P[i] = q * np.minimum(1.0, (pi / q) / (pi[i] / q[i]))
        P[i, i] = 0.0
        P[i, i] = 1.0 - P[i].sum()
    return P


def markov_chi2(counts: np.ndarray, pi: np.ndarray, q: np.ndarray | None = None) -> tuple[float, int, float]:
    """(statistic, dof, p-value) of the chain-CLT chi-square on the support.
    q: the alias proposal's probabilities over all candidates (None: uniform)."""
    sup = pi > 0
    pi_s = pi[sup] / pi[sup].sum()
    c = counts[sup].astype(np.float64)
    if counts[~sup].sum() > 0:
        return float("inf"), 0, 0.0  # zero-weight candidate emitted
    n = len(pi_s)
    if n < 2:
        return 0.0, 0, 1.0
    P = mh_kernel(pi_s, proposals=len(pi), q=None if q is None else q[sup] / q.sum())
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


def audit(g: O.HostGraph, oracle: O.Oracle, md: O.ModelDesc, rows, lens, min_visits=5000, max_states=40,
          alias_proposal=False):
    """p-values of the chain chi-square for states visited >= min_visits
    (alias_proposal: the chains ran the static-weight alias proposal)."""
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
        q = g.w[int(g.offsets[v]):int(g.offsets[v + 1])].astype(np.float64) if alias_proposal else None
        pv.append(markov_chi2(counts, pi, q)[2])
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


def lumped_chi2(counts: np.ndarray, pi: np.ndarray) -> tuple[float, int, float]:
    """The chain-CLT chi-square after lumping candidates of equal target
    weight. Under the uniform-proposal kernel, P(i -> class B) =
    (|B| / m) min(1, pi_B / pi_i) is the same for every i of a class A, so the
    class sequence is itself an exact Markov chain (strong lumpability) and the
    test needs a matrix of (distinct weights) x (distinct weights) only --
    3 x 3 for unweighted node2vec however large the hub. Zero-weight
    candidates are proposed (m = all candidates) and never accepted."""
    m = len(pi)
    if counts[pi <= 0].sum() > 0:
        return float("inf"), 0, 0.0
    vals, inv = np.unique(pi[pi > 0], return_inverse=True)
    c = np.bincount(inv, weights=counts[pi > 0].astype(np.float64), minlength=len(vals))
    size = np.bincount(inv, minlength=len(vals)).astype(np.float64)
    k = len(vals)
    if k < 2:
        return 0.0, 0, 1.0
    Pi = size * vals
    Pi = Pi / Pi.sum()
    P = np.zeros((k, k))
    for a in range(k):
        P[a] = size / m * np.minimum(1.0, vals / vals[a])
        P[a, a] = 0.0
        P[a, a] = 1.0 - P[a].sum()
    Z = np.linalg.inv(np.eye(k) - P + np.outer(np.ones(k), Pi))
    D = np.diag(Pi)
    S = D @ Z + Z.T @ D - D - np.outer(Pi, Pi)
    N = c.sum()
    d = c / N - Pi
    stat = float(N * d @ np.linalg.pinv(S, rcond=1e-10, hermitian=True) @ d)
    return stat, k - 1, float(st.chi2.sf(stat, k - 1))


def transition_counts_gpu(rows, lens, kind, offsets, nbr, metapath=None, min_visits=5000, max_states=40,
                          max_support=None, max_classes=None, pi_classes=None):
    """Per-state next-node counts of a (large) corpus, counted on the GPU
    with torch (test infrastructure only). States as `transitions`: deepwalk
    v; metapath2vec (v, required type); second order the arc (v -> prev),
    i.e. state (prev, v) with affix = index of prev in N(v). Returns a list of
    (v, affix, visits, counts over N(v)) for the `max_states` most visited
    states with >= min_visits visits (and degree <= max_support if given)."""
    import torch
    dev = torch.device("cuda" if torch.cuda.is_available() else "cpu")
    off = torch.from_numpy(np.asarray(offsets, dtype=np.int64)).to(dev)
    n = off.numel() - 1
    deg = off[1:] - off[:-1]
    src = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int64), deg)
    arckey = (src << 32) | torch.from_numpy(np.asarray(nbr, dtype=np.int64)).to(dev)
    del src
    R = torch.from_numpy(np.ascontiguousarray(rows).view(np.int32)).to(dev)
    Ln = torch.from_numpy(np.asarray(lens, dtype=np.int64)).to(dev)
    S = R.shape[1]
    second = kind in (O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK)
    first_col = 1 if second else 0
    cols = torch.arange(first_col, S - 1, device=dev)
    valid = (cols[None, :] + 1) < Ln[:, None]
    cur = R[:, first_col:S - 1][valid].long()
    nxt = R[:, first_col + 1:S][valid].long()
    if second:
        prev = R[:, first_col - 1:S - 2][valid].long()
        sid = torch.searchsorted(arckey, (cur << 32) | prev)
        n_states = arckey.numel()
    elif kind == O.METAPATH2VEC:
        T = int(max(metapath)) + 1
        req = np.zeros(S, dtype=np.int64)
        a = 0
        for i in range(S):
            req[i] = metapath[_next(a, metapath)]
            a = _next(a, metapath)
        reqc = torch.from_numpy(req).to(dev)[cols]
        sid = cur * T + reqc[None, :].expand_as(valid)[valid]
        n_states = n * T
    else:
        sid = cur
        n_states = n
    del R
    visits = torch.bincount(sid, minlength=n_states)
    # node of each state and its support
    if second:
        node = torch.arange(n_states, device=dev)
        node = torch.searchsorted(off[1:], node, right=True)
    elif kind == O.METAPATH2VEC:
        node = torch.arange(n_states, device=dev) // T
    else:
        node = torch.arange(n_states, device=dev)
    ok = visits >= min_visits
    if max_support is not None:
        ok &= deg[node] <= max_support
    cand = torch.nonzero(ok).flatten()
    order = torch.argsort(visits[cand], descending=True)[:max_states]
    chosen = cand[order]
    flag = torch.full((n_states,), -1, dtype=torch.int64, device=dev)
    flag[chosen] = torch.arange(chosen.numel(), device=dev)
    sel = flag[sid]
    m = sel >= 0
    # counts per (chosen state, candidate index): several chosen states can
    # share a node v (second order: (s1, v) and (s2, v)), so the cell is keyed
    # by the state as well as by the arc v -> next
    cell = torch.searchsorted(arckey, (cur[m] << 32) | nxt[m]) - off[cur[m]]
    dmax = int(deg[node[chosen]].max()) if chosen.numel() else 1
    cnt = torch.bincount(sel[m] * dmax + cell, minlength=max(1, chosen.numel() * dmax))
    out = []
    offs = np.asarray(offsets, dtype=np.int64)
    for i, (st_id, vis) in enumerate(zip(chosen.tolist(), visits[chosen].tolist())):
        v = int(node[st_id])
        if second:
            aff = int(st_id - offs[v])
        elif kind == O.METAPATH2VEC:
            r = st_id % T
            aff = next(a for a in range(len(metapath)) if metapath[_next(a, metapath)] == r)
        else:
            aff = O.NO_AFFIX
        out.append((v, aff, vis, cnt[i * dmax:i * dmax + int(offs[v + 1] - offs[v])].cpu().numpy()))
    return out


def min_class_entries(pi: np.ndarray, visits: int) -> float:
    """Smallest expected number of entries, over `visits` transitions, into a
    class of equal target weight of a uniform-proposal chain (stationary
    entries into B per step = Pi_B (1 - P_BB)). The chain CLT behind the test
    needs many of them: a hub state whose heavy class is one candidate among
    20,000 is entered about once per 20,000 proposals, so at 5,000-10,000
    visits its count is a Poisson number of excursions, not Gaussian -- any
    correct implementation then scores heavy-tailed p-values (SURVEY 8(c):
    "expected cell >= 5")."""
    vals, inv = np.unique(pi[pi > 0], return_inverse=True)
    size = np.bincount(inv, minlength=len(vals)).astype(np.float64)
    k, m = len(vals), len(pi)
    if k < 2:
        return float("inf")
    Pi = size * vals / np.sum(size * vals)
    out = []
    for a in range(k):
        stay = 1.0 - np.sum(np.delete(size / m * np.minimum(1.0, vals / vals[a]), a))
        out.append(visits * Pi[a] * (1.0 - stay))
    return float(min(out))


def audit_counts(g: O.HostGraph, oracle: O.Oracle, md: O.ModelDesc, states, dense_max=1024, min_entries=None):
    """p-values of the chain chi-square of (v, affix, visits, counts) states:
    the full test up to dense_max candidates, the lumped (equal target weight)
    test beyond, where the distinct weights are few. min_entries: audit a
    lumped state only if every weight class is expected to be entered at
    least that often (min_class_entries)."""
    pv = []
    for v, aff, vis, counts in states:
        pi = O.eval_target(g, oracle, md, v, aff)
        assert counts.sum() == vis
        # (the guard applies to the lumped test: its classes can be single,
        # sticky candidates at hubs; the dense test's cells are candidates)
        if min_entries is not None and len(pi) > dense_max and min_class_entries(pi, vis) < min_entries:
            continue
        if len(pi) <= dense_max:
            pv.append(markov_chi2(counts, pi)[2])
        else:
            pv.append(lumped_chi2(counts, pi)[2])
    return np.array(pv)
