"""Sparse / dense attention operators (reference pkg/src/dynsparse/attention.py).

Same names, argument meaning and error behaviour as the reference:
  * CriticalIndexSet          attention.py:31-78  (sorted, unique, non-negative rows)
  * full_attention            attention.py:95-109
  * sparse_attention          attention.py:153-187 (softmax renormalised over the
                              selected keys; every query needs >= 1 key)
  * head_sparsity             attention.py:143-150
Host (numpy) float inputs run on the CUDA-core CSR kernels in fp32 (the
precision path); group-tiled bf16 work runs on the tcgen05 kernels
(grouping.grouped_sparse_attention, layer.DSVAttentionLayer).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _convert as cv
from . import ops


def _check_unit_interval(name: str, value: float, *, open_low=False, open_high=False) -> float:
    value = float(value)
    low_ok = value > 0.0 if open_low else value >= 0.0
    high_ok = value < 1.0 if open_high else value <= 1.0
    if not (low_ok and high_ok and np.isfinite(value)):
        lo = "(" if open_low else "["
        hi = ")" if open_high else "]"
        raise ValueError(f"{name} must lie in {lo}0, 1{hi}, got {value}")
    return value


@dataclass
class CriticalIndexSet:
    """Per-query selected KV indices (attention.py:31-78)."""

    indices: list
    theta: float | None = None

    def __post_init__(self):
        if self.theta is not None:
            self.theta = _check_unit_interval("theta", self.theta, open_low=True)
        cleaned = []
        for q, idx in enumerate(self.indices):
            idx = np.asarray(idx.cpu() if isinstance(idx, torch.Tensor) else idx, dtype=np.int64)
            if idx.ndim != 1:
                raise ValueError(f"index list for query {q} must be 1D")
            if idx.size and (np.any(np.diff(idx) <= 0) or idx[0] < 0):
                raise ValueError(f"indices for query {q} must be sorted, unique, nonnegative")
            cleaned.append(idx)
        self.indices = cleaned

    @property
    def n_queries(self) -> int:
        return len(self.indices)

    def sizes(self) -> np.ndarray:
        return np.array([idx.size for idx in self.indices], dtype=np.int64)

    def total_pairs(self) -> int:
        return int(self.sizes().sum())

    def uniform_k(self) -> int | None:
        sizes = self.sizes()
        if sizes.size and np.all(sizes == sizes[0]):
            return int(sizes[0])
        return None

    def as_array(self) -> np.ndarray:
        k = self.uniform_k()
        if k is None:
            raise ValueError("index set is ragged; no uniform (S, k) form")
        return np.stack(self.indices) if k else np.empty((self.n_queries, 0), np.int64)

    def to_csr(self, device=None):
        """(ptr int64 [S+1], cols int32) on `device` — the CSR form the kernels read."""
        sizes = self.sizes()
        ptr = np.zeros(sizes.size + 1, dtype=np.int64)
        np.cumsum(sizes, out=ptr[1:])
        cols = (np.concatenate(self.indices) if self.indices else np.empty(0, np.int64)).astype(np.int32)
        dev = device or cv.device()
        return torch.from_numpy(ptr).to(dev), torch.from_numpy(cols).to(dev)


def _prep_qk(q, k):
    q = cv.as_matrix("Q", q)
    k = cv.as_matrix("K", k)
    cv.check_same_cols("Q", q, "K", k)
    return q, k


def _compute_dtype(x):
    if cv.is_torch(x) and x.dtype == torch.bfloat16:
        return torch.bfloat16
    return torch.float32


def _out_dtype(x):
    return x.dtype if not cv.is_torch(x) else None


def full_attention(q, k, v, *, flops=None):
    """softmax(Q K^T / sqrt(d_k)) V (attention.py:95-109), all keys per query."""
    q, k = _prep_qk(q, k)
    v = cv.as_matrix("V", v)
    if v.shape[0] != k.shape[0]:
        raise ValueError(f"V has {v.shape[0]} rows but K has {k.shape[0]}")
    if v.shape[1] != q.shape[1]:
        raise ValueError("the device kernels need d_v == d_k")
    dt = _compute_dtype(q)
    tq, tk, tv = (cv.to_device(t, dt).unsqueeze(0) for t in (q, k, v))
    out, _ = ops.rows_fwd(tq, tk, tv, None, None, scale=1.0 / math.sqrt(q.shape[1]))
    if flops is not None:
        flops.add_pairs(q.shape[0] * k.shape[0], q.shape[1])
        flops.add_per_query(q.shape[0])
    return cv.back(out[0], q, _out_dtype(q))


def sparse_attention(q, k, v, idx: CriticalIndexSet, *, flops=None):
    """Attention restricted to each query's selected keys (attention.py:153-187)."""
    q, k = _prep_qk(q, k)
    v = cv.as_matrix("V", v)
    if idx.n_queries != q.shape[0]:
        raise ValueError(f"index set covers {idx.n_queries} queries, Q has {q.shape[0]}")
    sizes = idx.sizes()
    if np.any(sizes == 0):
        raise ValueError("every query needs at least one selected index")
    if v.shape[1] != q.shape[1]:
        raise ValueError("the device kernels need d_v == d_k")
    if idx.total_pairs() and max(int(i.max()) for i in idx.indices if i.size) >= k.shape[0]:
        raise ValueError("index set references keys beyond K")
    dt = _compute_dtype(q)
    tq, tk, tv = (cv.to_device(t, dt).unsqueeze(0) for t in (q, k, v))
    ptr, cols = idx.to_csr(tq.device)
    out, _ = ops.rows_fwd(tq, tk, tv, ptr, cols, scale=1.0 / math.sqrt(q.shape[1]))
    if flops is not None:
        flops.add_pairs(idx.total_pairs(), q.shape[1])
        flops.add_per_query(q.shape[0])
    return cv.back(out[0], q, _out_dtype(q))


def head_sparsity(idx: CriticalIndexSet, s_total: int) -> float:
    """Mean non-critical fraction (attention.py:143-150)."""
    if s_total < 1:
        raise ValueError("s_total must be positive")
    sizes = idx.sizes()
    if np.any(sizes > s_total):
        raise ValueError("index set references more keys than s_total")
    return float(np.mean((s_total - sizes) / s_total))
