"""Host-side walker partitioning for multi-GPU runs.

Walkers are independent, so the only multi-GPU structure is a partition of
the walker index range (v-major, k-minor, engine.cpp:179-185) into contiguous
start-node ranges, one per device, each device holding a full CSR replica and
a private chain table. Ranges are cut at equal active-walker counts (equal id
ranges leave R-MAT's isolated high ids unbalanced). The corpus is
the concatenation of the per-device corpora in device order, which is the
reference's corpus order (engine.cpp:220-226).
"""
from __future__ import annotations

import numpy as np


def active_nodes(degrees: np.ndarray, valid: np.ndarray | None = None) -> np.ndarray:
    """Start nodes that run walkers: valid start and degree > 0."""
    act = degrees > 0
    if valid is not None:
        act &= valid
    return np.nonzero(act)[0]


def balanced_cuts(degrees: np.ndarray, parts: int, valid: np.ndarray | None = None) -> np.ndarray:
    """cuts[0] = 0, cuts[parts] = n; range i = [cuts[i], cuts[i+1]). Cut i
    starts at the active node of rank floor(i * n_act / parts) -- the rule of
    mhw_partition_nodes (walk.cu partition_nodes)."""
    n = len(degrees)
    act = active_nodes(degrees, valid)
    cuts = np.full(parts + 1, n, dtype=np.int64)
    cuts[0] = 0
    for i in range(1, parts):
        r = i * len(act) // parts
        cuts[i] = act[r] if r < len(act) else n
        cuts[i] = max(cuts[i], cuts[i - 1])
    return cuts


def rows_in_range(cuts: np.ndarray, rank: int, K: int, valid: np.ndarray | None, n: int) -> tuple[int, int]:
    """[first, last) corpus rows owned by `rank` (valid starts emit K rows)."""
    v = np.ones(n, dtype=bool) if valid is None else valid
    before = int(np.sum(v[:cuts[rank]])) * K
    mine = int(np.sum(v[cuts[rank]:cuts[rank + 1]])) * K
    return before, before + mine


def imbalance(degrees: np.ndarray, cuts: np.ndarray, valid: np.ndarray | None = None) -> float:
    """max / mean active walkers per part."""
    act = np.zeros(len(degrees), dtype=np.int64)
    act[active_nodes(degrees, valid)] = 1
    per = np.array([act[cuts[i]:cuts[i + 1]].sum() for i in range(len(cuts) - 1)], dtype=np.float64)
    return float(per.max() / per.mean()) if per.mean() > 0 else 1.0
