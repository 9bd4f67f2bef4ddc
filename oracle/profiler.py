"""Oracle: sampled sparsity profiler (test infrastructure only; see oracle/__init__.py).

Restates pkg/src/dynsparse/profiler.py and attention.py:
  * sample_queries          profiler.py:33-45   ceil(S / factor) distinct rows, uniform,
                                                 default_rng(seed), sorted
  * critical_counts         attention.py:118-140 shortest descending-score prefix (ties toward
                                                 the lower index) reaching min(theta, csum[-1])
                                                 - 1e-9 of the row's softmax mass
  * measure_block_sparsity  profiler.py:48-79   logits = q[rows] k^T / sqrt(d), max-shifted
                                                 softmax in fp64, head_sparsity
                                                 (attention.py:143-150) of the oracle sets
"""

from __future__ import annotations

import numpy as np

MASS_EPS = 1e-9   # attention.py:28


def sample_queries(s_total: int, factor: int, seed: int) -> np.ndarray:
    """profiler.py:33-45."""
    if s_total < 1:
        raise ValueError("s_total must be positive")
    if s_total < factor:
        raise ValueError(f"need S >= factor, got S={s_total}, factor={factor}")
    n = int(np.ceil(s_total / factor))
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(s_total, size=n, replace=False))


def critical_counts(scores: np.ndarray, theta: float) -> np.ndarray:
    """Per-row |I_q| of attention.py:118-140 on post-softmax rows."""
    scores = np.asarray(scores, dtype=np.float64)
    out = np.empty(scores.shape[0], dtype=np.int64)
    cols = np.arange(scores.shape[1])
    for r, row in enumerate(scores):
        order = np.lexsort((cols, -row))
        csum = np.cumsum(row[order])
        target = min(theta, csum[-1]) - MASS_EPS
        out[r] = min(int(np.searchsorted(csum, target, side="left")) + 1, row.size)
    return out


def softmax_rows(logits: np.ndarray) -> np.ndarray:
    """profiler.py:74-77: shift by the row max, exp, normalise (fp64)."""
    logits = np.asarray(logits, dtype=np.float64)
    logits = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(logits)
    return e / e.sum(axis=1, keepdims=True)


def measure_block_sparsity(qs, ks, theta: float, factor: int, seed: int) -> np.ndarray:
    """profiler.py:48-79 (per head: sampled rows, softmax, oracle sets, head_sparsity)."""
    s_total = np.asarray(qs[0]).shape[0]
    rows = sample_queries(s_total, factor, seed)
    vals = np.empty(len(qs))
    for h, (q, k) in enumerate(zip(qs, ks)):
        q = np.asarray(q, dtype=np.float64)
        k = np.asarray(k, dtype=np.float64)
        p = softmax_rows(q[rows] @ k.T / np.sqrt(q.shape[1]))
        sizes = critical_counts(p, theta)
        vals[h] = float(np.mean((s_total - sizes) / s_total))
    return vals
