"""Critical-KV top-k selection (reference pkg/src/dynsparse/selection.py).

`streaming_topk` / `twopass_select` keep the reference signatures and exact
semantics — per query the k largest scores of Q_lr K_lr^T, ties toward the lower
key index, indices ascending, threshold = k-th largest score — but run on the
GPU in row chunks, so the S x S product is only ever materialised one chunk at a
time (within the reference's O(S k) working set). Host (numpy) and torch fp64
inputs take the reference-precision path: fp64 score tiles (dsv_gemm_f64) and the
fp64 top-k (dsv_topk_f64), fp64 thresholds. torch fp32 / bf16 inputs score in
fp32 (deterministic t-order fmaf) and select with the K2 kernel. Given identical
scores the selected sets are bit-exact with the reference rule
(tests/test_gpu_api.py, tests/test_gpu_kernels.py, conformance/).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _convert as cv
from . import ops
from .attention import CriticalIndexSet

DEFAULT_TILE = 128
_ROW_CHUNK_BYTES = 1 << 30   # score scratch per chunk


@dataclass
class AllocationMeter:
    """Counts live auxiliary entries (selection.py:31-45). The device path
    materialises one score chunk plus the (S, k) result, both recorded here."""

    current: int = 0
    peak: int = 0
    events: list = field(default_factory=list)

    def grab(self, n_entries: int, label: str = "") -> None:
        self.current += int(n_entries)
        self.peak = max(self.peak, self.current)
        self.events.append((label, int(n_entries)))

    def release(self, n_entries: int) -> None:
        self.current -= int(n_entries)


@dataclass
class TopKResult:
    """Exact per-query top-k: (S, k) ascending indices + k-th scores (selection.py:48-57)."""

    indices: np.ndarray
    thresholds: np.ndarray
    k: int

    def to_index_set(self) -> CriticalIndexSet:
        return CriticalIndexSet(list(np.asarray(self.indices)), theta=None)


def k_from_sparsity(sparsity: float, s_total: int) -> int:
    """selection.py:60-67: max(1, ceil((1 - sparsity) * S))."""
    sparsity = float(sparsity)
    if not 0.0 <= sparsity < 1.0:
        raise ValueError(f"sparsity must lie in [0, 1), got {sparsity}")
    if s_total < 1:
        raise ValueError("s_total must be positive")
    return max(1, int(math.ceil((1.0 - sparsity) * s_total)))


def _prep(q_lr, k_lr, k):
    q_lr = cv.as_matrix("Q_lr", q_lr)
    k_lr = cv.as_matrix("K_lr", k_lr)
    cv.check_same_cols("Q_lr", q_lr, "K_lr", k_lr)
    k = int(k)
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    if k > k_lr.shape[0]:
        raise ValueError(f"k={k} exceeds the {k_lr.shape[0]} available keys")
    return q_lr, k_lr, k


def _chunk_rows(s_q: int, s_k: int, k_max: int, elem: int) -> int:
    """Score rows per chunk: the live score chunk stays within 4 S k entries (the reference's
    O(S k) working-set contract, selection.py:31-45 / tests/test_selection.py:100-107:
    peak <= 8 S k with the (S, k) results) and within _ROW_CHUNK_BYTES."""
    return max(1, min(s_q, (4 * s_q * k_max) // s_k, _ROW_CHUNK_BYTES // (elem * s_k)))


def topk_scores_device(q: torch.Tensor, kk: torch.Tensor, k_per_row, meter=None, flops=None,
                       return_scores: bool = False):
    """Exact top-k of q @ kk.T on device; k_per_row: int or int tensor [S_q].

    q: [S_q, r], kk: [S_k, r] CUDA tensors: fp64 (the reference-precision path: fp64 score
    tiles on dsv_gemm_f64, fp64 top-k, fp64 thresholds) or fp32 / bf16 (fp32 scores, K2).
    Returns (idx int32 [S_q, k_max], thr [S_q]) and optionally the score matrix.
    """
    s_q, r = q.shape
    s_k = kk.shape[0]
    f64 = q.dtype == torch.float64
    sdt = torch.float64 if f64 else torch.float32
    if isinstance(k_per_row, int):
        kvec = torch.full((1,), k_per_row, dtype=torch.int32, device=q.device)
        rows_per = max(s_q, 1)
        k_max = k_per_row
    else:
        kvec = k_per_row.to(device=q.device, dtype=torch.int32)
        rows_per = 1
        k_max = int(kvec.max().item())
    idx = torch.empty((s_q, k_max), dtype=torch.int32, device=q.device)
    thr = torch.empty((s_q,), dtype=sdt, device=q.device)
    all_scores = torch.empty((s_q, s_k), dtype=sdt, device=q.device) if return_scores else None
    chunk = _chunk_rows(s_q, s_k, k_max, 8 if f64 else 4)
    if meter is not None:
        meter.grab(2 * s_q * k_max, "result buffers")
    buf = None
    for r0 in range(0, s_q, chunk):
        r1 = min(r0 + chunk, s_q)
        if all_scores is not None:
            sc = all_scores[r0:r1]
        else:
            if buf is None:
                buf = torch.empty((chunk, s_k), dtype=sdt, device=q.device)
            sc = buf[: r1 - r0]
        if f64:
            ops.gemm_f64(q[r0:r1], kk.t(), out=sc)
        else:
            ops.scores_f32(q[r0:r1], kk, out=sc.unsqueeze(0))
        if meter is not None:
            meter.grab(sc.numel(), "score chunk")
        kv = kvec if rows_per != 1 else kvec[r0:r1]
        rp = rows_per if rows_per != 1 else 1
        if f64:
            ii, tt = ops.topk_f64(sc, kv, rp, k_max)
        else:
            ii, tt = ops.topk_rows(sc, kv, rp, k_max)
        idx[r0:r1] = ii
        thr[r0:r1] = tt
        if meter is not None:
            meter.release(sc.numel())
        if flops is not None:
            flops.estimation += (r1 - r0) * s_k * 2 * r
            flops.selection += (r1 - r0) * s_k
    if meter is not None:
        meter.release(2 * s_q * k_max)
    return (idx, thr, all_scores) if return_scores else (idx, thr)


def _run(q_lr, k_lr, k, meter=None, flops=None) -> TopKResult:
    q_lr, k_lr, k = _prep(q_lr, k_lr, k)
    if cv.wants_f64(q_lr) and cv.wants_f64(k_lr):
        dt = torch.float64
    elif cv.is_torch(q_lr) and q_lr.dtype == torch.bfloat16:
        dt = torch.bfloat16
    else:
        dt = torch.float32
    qd, kd = cv.to_device(q_lr, dt), cv.to_device(k_lr, dt)
    idx, thr = topk_scores_device(qd, kd, k, meter=meter, flops=flops)
    if cv.is_torch(q_lr):
        return TopKResult(indices=idx.long(), thresholds=thr.double(), k=k)
    return TopKResult(indices=idx.cpu().numpy().astype(np.int64),
                      thresholds=thr.cpu().numpy().astype(np.float64), k=k)


def streaming_topk(q_lr, k_lr, k: int, *, tile: int = DEFAULT_TILE, meter: AllocationMeter | None = None,
                   flops=None) -> TopKResult:
    """Exact per-query top-k of Q_lr K_lr^T (selection.py:118-175).

    `tile` is accepted for signature compatibility; like the reference it has no
    semantic effect (the device kernels tile internally).
    """
    del tile
    return _run(q_lr, k_lr, k, meter=meter, flops=flops)


def twopass_select(q_lr, k_lr, k: int, *, tile: int = DEFAULT_TILE, flops=None) -> TopKResult:
    """Threshold-then-gather selection (selection.py:178-242); the K2 kernel is this
    two-pass scheme (k-th key, then ordered '>' / '==' compaction), so the result is
    identical to streaming_topk."""
    del tile
    return _run(q_lr, k_lr, k, flops=flops)
