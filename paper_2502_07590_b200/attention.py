"""Sparse / dense attention operators (reference pkg/src/dynsparse/attention.py).

Same names, argument meaning and error behaviour as the reference:
  * CriticalIndexSet          attention.py:31-78  (sorted, unique, non-negative rows)
  * full_attention            attention.py:95-109
  * sparse_attention          attention.py:153-187 (softmax renormalised over the
                              selected keys; every query needs >= 1 key)
  * head_sparsity             attention.py:143-150
  * attention_scores          attention.py:112-115
  * critical_kv_oracle        attention.py:118-140 (theta-mass prefix, ties -> lower index)
  * analyze_distribution      attention.py:190-253
Host (numpy) and torch fp64 inputs run the fp64 kernels (precise.cu, rows_simt.cu:
the reference computes in the caller's dtype); torch fp32 / bf16 inputs the fp32
CUDA-core CSR kernels; group-tiled bf16 work the tcgen05 kernels
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


_MASS_EPS = 1e-9


def _prep_qk(q, k):
    q = cv.as_matrix("Q", q)
    k = cv.as_matrix("K", k)
    cv.check_same_cols("Q", q, "K", k)
    return q, k


def _compute_dtype(*xs):
    """Reference precision for host / fp64 inputs (fp64 kernels); torch bf16 runs the
    bf16-input fp32 kernels, torch fp32 the fp32 kernels."""
    if all(cv.wants_f64(x) for x in xs):
        return torch.float64
    if cv.is_torch(xs[0]) and xs[0].dtype == torch.bfloat16:
        return torch.bfloat16
    return torch.float32


def _out_dtype(x):
    return x.dtype if not cv.is_torch(x) else None


def _attend(q, k, v, ptr, cols):
    """Row attention on the device in the compute dtype; returns (out, dtype) with out on the
    device (fp64 kernels for the precision path, fp32 CUDA-core kernels otherwise)."""
    dt = _compute_dtype(q, k, v)
    tq, tk, tv = (cv.to_device(t, dt).unsqueeze(0) for t in (q, k, v))
    if dt == torch.float64:
        out, _ = ops.rows_fwd_f64(tq, tk, tv, ptr, cols, 1.0 / math.sqrt(q.shape[1]))
    else:
        if v.shape[1] != q.shape[1]:
            raise ValueError("the fp32 / bf16 device kernels need d_v == d_k")
        out, _ = ops.rows_fwd(tq, tk, tv, ptr, cols, scale=1.0 / math.sqrt(q.shape[1]))
    return out[0]


def full_attention(q, k, v, *, flops=None):
    """softmax(Q K^T / sqrt(d_k)) V (attention.py:95-109), all keys per query."""
    q, k = _prep_qk(q, k)
    v = cv.as_matrix("V", v)
    if v.shape[0] != k.shape[0]:
        raise ValueError(f"V has {v.shape[0]} rows but K has {k.shape[0]}")
    out = _attend(q, k, v, None, None)
    if flops is not None:
        flops.add_pairs(q.shape[0] * k.shape[0], q.shape[1])
        flops.add_per_query(q.shape[0])
    return cv.back(out, q, cv.result_dtype(q, k, v))


def attention_scores(q, k):
    """Post-softmax score matrix softmax(Q K^T / sqrt(d)) (attention.py:112-115): fp64 logits
    (dsv_gemm_f64, divided by sqrt(d)) and the max-subtracted row softmax on the device."""
    q, k = _prep_qk(q, k)
    dt = _compute_dtype(q, k)
    qd, kd = cv.to_device(q, torch.float64), cv.to_device(k, torch.float64)
    sc = ops.gemm_f64(qd, kd.t(), div=float(np.sqrt(q.shape[1])))
    ops.softmax_rows_f64_(sc)
    if cv.is_torch(q):
        return sc if dt == torch.float64 else sc.to(q.dtype)
    return cv.back(sc, q, cv.result_dtype(q, k))


def _critical_device(sc: torch.Tensor, theta: float) -> list:
    """Per row of fp64 post-softmax scores: the minimal descending-score prefix (ties toward
    the lower index) whose mass reaches min(theta, total) - 1e-9, as sorted index arrays.
    Prefix length: dsv_sorted_stats_f64 (sorted row, sequential cumsum); the set itself: the
    exact top-n_keep of the row (dsv_topk_f64 with per-row k, the same order)."""
    n_keep, _ = ops.sorted_stats_f64(sc, theta=theta, eps=_MASS_EPS)
    kmax = int(n_keep.max().item())
    idx, _ = ops.topk_f64(sc, n_keep, 1, kmax)
    nk = n_keep.cpu().numpy()
    ii = idx.cpu().numpy()
    return [ii[r, : nk[r]].astype(np.int64) for r in range(sc.shape[0])]


def critical_kv_oracle(scores, theta: float) -> CriticalIndexSet:
    """Minimal descending-score prefix reaching cumulative mass theta (attention.py:118-140)."""
    theta = _check_unit_interval("theta", theta, open_low=True)
    scores = cv.as_matrix("scores", scores)
    if bool((scores < 0).any()):
        raise ValueError("scores must be nonnegative (post-softmax)")
    sc = cv.to_device(scores, torch.float64)
    return CriticalIndexSet(_critical_device(sc, theta), theta=theta)


def analyze_distribution(scores, grid=None, *, theta: float = 0.9, top_fraction: float = 0.1,
                         mass_threshold: float = 0.9, n_bins: int = 50) -> dict:
    """Score-distribution statistics over a post-softmax matrix (attention.py:190-253): the
    top-fraction mass per row (sorted on the device, dsv_sorted_stats_f64), a log-spaced
    histogram (dsv_histogram_f64, np.histogram semantics), and with a grid the distance
    statistics of the theta-critical keys (critical_kv_oracle on the device)."""
    scores = cv.as_matrix("scores", scores)
    s_total = scores.shape[1]
    top_n = max(1, int(np.ceil(top_fraction * s_total)))
    sc = cv.to_device(scores, torch.float64)
    _, top_mass = ops.sorted_stats_f64(sc, top_n=top_n, want_keep=False, want_top=True)
    top_mass = top_mass.cpu().numpy()
    concentrated = float(np.mean(top_mass >= mass_threshold - _MASS_EPS))
    pos = sc[sc > 0]
    lo = max(float(pos.min().item()), 1e-12) if pos.numel() else 1e-12
    edges = np.logspace(np.log10(lo), 0.0, n_bins + 1)
    hist = ops.histogram_f64(sc, torch.from_numpy(edges).to(sc.device)).cpu().numpy()
    report = {
        "n_queries": int(scores.shape[0]), "n_keys": int(s_total),
        "top_fraction": float(top_fraction), "mass_threshold": float(mass_threshold),
        "top_mass_fraction_mean": float(top_mass.mean()),
        "concentrated_query_fraction": concentrated,
        "histogram": {"edges": edges.tolist(), "counts": hist.tolist()},
    }
    if grid is not None:
        if grid.size != s_total or scores.shape[0] != s_total:
            raise ValueError(f"grid distance statistics need square S x S scores with "
                             f"S = {grid.size}, got {tuple(scores.shape)}")
        if bool((sc < 0).any()):
            raise ValueError("scores must be nonnegative (post-softmax)")
        theta = _check_unit_interval("theta", theta, open_low=True)
        sets = _critical_device(sc, theta)
        coords = grid.coords_array().astype(np.float64)
        per_query = np.empty(len(sets))
        within5 = beyond10 = total = 0
        for row, sel in enumerate(sets):
            d = np.linalg.norm(coords[sel] - coords[row], axis=1)
            per_query[row] = d.mean()
            within5 += int(np.sum(d <= 5.0))
            beyond10 += int(np.sum(d > 10.0))
            total += sel.size
        report["critical_kv"] = {"theta": float(theta), "mean_distance": float(per_query.mean()),
                                 "fraction_within_radius_5": within5 / total,
                                 "fraction_beyond_radius_10": beyond10 / total}
    return report


def sparse_attention(q, k, v, idx: CriticalIndexSet, *, flops=None):
    """Attention restricted to each query's selected keys (attention.py:153-187)."""
    q, k = _prep_qk(q, k)
    v = cv.as_matrix("V", v)
    if idx.n_queries != q.shape[0]:
        raise ValueError(f"index set covers {idx.n_queries} queries, Q has {q.shape[0]}")
    sizes = idx.sizes()
    if np.any(sizes == 0):
        raise ValueError("every query needs at least one selected index")
    if v.shape[0] != k.shape[0]:
        raise ValueError(f"V has {v.shape[0]} rows but K has {k.shape[0]}")
    if idx.total_pairs() and max(int(i.max()) for i in idx.indices if i.size) >= k.shape[0]:
        raise IndexError("index set references keys beyond K")
    ptr, cols = idx.to_csr(cv.device())
    out = _attend(q, k, v, ptr, cols)
    if flops is not None:
        flops.add_pairs(idx.total_pairs(), q.shape[1])
        flops.add_per_query(q.shape[0])
    return cv.back(out, q, cv.result_dtype(q, k, v))


def head_sparsity(idx: CriticalIndexSet, s_total: int) -> float:
    """Mean non-critical fraction (attention.py:143-150)."""
    if s_total < 1:
        raise ValueError("s_total must be positive")
    sizes = idx.sizes()
    if np.any(sizes > s_total):
        raise ValueError("index set references more keys than s_total")
    return float(np.mean((s_total - sizes) / s_total))
