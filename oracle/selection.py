"""Oracle: exact top-k selection (test infrastructure only; see oracle/__init__.py).

Restates pkg/src/dynsparse/selection.py:
  * k_from_sparsity           selection.py:60-67   max(1, ceil((1 - s) * S))
  * tie rule / emit order     selection.py:82-115 (_merge_block: keep > v*, then the
                              lowest-index entries == v*), :166-174 (ascending emit,
                              threshold = min kept score), :178-242 (twopass_select:
                              k-th value pass, then '>' plus the first '==' in index order)
numpy's `==` / `>` treat -0.0 and +0.0 as equal, and so does this oracle.
"""

from __future__ import annotations

import math

import numpy as np


def k_from_sparsity(sparsity: float, s_total: int) -> int:
    """selection.py:60-67."""
    sparsity = float(sparsity)
    if not 0.0 <= sparsity < 1.0:
        raise ValueError(f"sparsity must lie in [0, 1), got {sparsity}")
    if s_total < 1:
        raise ValueError("s_total must be positive")
    return max(1, int(math.ceil((1.0 - sparsity) * s_total)))


def topk_from_scores(scores: np.ndarray, k) -> tuple[np.ndarray, np.ndarray]:
    """Exact per-row top-k of a score matrix (two-pass scheme, selection.py:178-242).

    ``k`` is an int or a per-row int array. Returns (indices int64 [R, k_max]
    ascending, with rows of smaller k padded by -1; thresholds float64 [R]).
    """
    s = np.asarray(scores)
    if s.ndim != 2:
        raise ValueError("scores must be 2-D")
    n_rows, n_cols = s.shape
    ks = np.broadcast_to(np.asarray(k, dtype=np.int64), (n_rows,))
    if np.any(ks < 1) or np.any(ks > n_cols):
        raise ValueError("k must lie in [1, S]")
    k_max = int(ks.max()) if n_rows else 0
    out = np.full((n_rows, k_max), -1, dtype=np.int64)
    thr = np.empty(n_rows, dtype=np.float64)
    for kv in np.unique(ks):
        rows = np.nonzero(ks == kv)[0]
        sub = s[rows]
        # pass 1: k-th largest value per row (selection.py:197-212)
        vstar = np.partition(sub, n_cols - kv, axis=1)[:, n_cols - kv]
        gt = sub > vstar[:, None]
        eq = sub == vstar[:, None]
        need = kv - gt.sum(axis=1)
        # pass 2: '>' plus the first `need` ties in index order (selection.py:214-241)
        keep = gt | (eq & (np.cumsum(eq, axis=1) <= need[:, None]))
        cols = np.nonzero(keep)[1].reshape(len(rows), kv)
        out[rows, :kv] = cols
        thr[rows] = vstar.astype(np.float64)
    return out, thr


def topk_lowrank(q_lr: np.ndarray, k_lr: np.ndarray, k: int):
    """streaming_topk(q_lr, k_lr, k) (selection.py:118-175) on fp64 scores."""
    scores = np.asarray(q_lr, dtype=np.float64) @ np.asarray(k_lr, dtype=np.float64).T
    return topk_from_scores(scores, k)
