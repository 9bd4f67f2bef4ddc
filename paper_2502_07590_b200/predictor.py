"""Low-rank critical-KV predictor (reference pkg/src/dynsparse/predictor.py).

Per attention block (the north_star: per head) two projections W_q, W_k in
R^{d x d_lr}; the predicted score matrix (X W_q)(X W_k)^T is ranked per query
and its top-k keys are the critical KV estimate. Here:
  * project            -> K1a tcgen05 GEMM (bf16 in, fp32 accumulate)
  * estimate_critical  -> K1a for both sides, then fp32 score rows (K1b) and the
                          exact K2 top-k; per-query k arrays use per-row k on
                          the device (same result as the reference's
                          top-k_max + re-rank, predictor.py:246-259, because the
                          top-k set of a row is nested in its top-k_max set).
The predictor training step (loss_and_grads / train_step, predictor.py:139-214)
is SURVEY §8(f) "next" work and is not part of this path yet.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _convert as cv
from . import ops
from .attention import CriticalIndexSet
from .selection import k_from_sparsity, topk_scores_device

COS_WEIGHT = 0.95
NORM_WEIGHT = 0.05


@dataclass
class PredictorParams:
    """Per-block projection matrices plus Adam state (predictor.py:38-83)."""

    w_q: np.ndarray
    w_k: np.ndarray
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    step: int = 0
    m_q: np.ndarray = None
    v_q: np.ndarray = None
    m_k: np.ndarray = None
    v_k: np.ndarray = None
    loss_history: list = field(default_factory=list)

    def __post_init__(self):
        self.w_q = np.asarray(cv.as_matrix("W_q", self.w_q))
        self.w_k = np.asarray(cv.as_matrix("W_k", self.w_k))
        if self.w_q.shape != self.w_k.shape:
            raise ValueError("W_q and W_k must share a shape")
        d, d_lr = self.w_q.shape
        if d_lr >= d:
            raise ValueError(f"low-rank width d_lr={d_lr} must be below d={d}")
        for name in ("m_q", "v_q", "m_k", "v_k"):
            if getattr(self, name) is None:
                setattr(self, name, np.zeros_like(self.w_q))
        self._dev = None

    @classmethod
    def initialize(cls, d: int, d_lr: int, seed: int = 0, lr: float = 1e-3) -> "PredictorParams":
        rng = np.random.default_rng(seed)
        scale = 1.0 / np.sqrt(d)
        return cls(w_q=rng.normal(0.0, scale, (d, d_lr)), w_k=rng.normal(0.0, scale, (d, d_lr)), lr=lr)

    @property
    def d(self) -> int:
        return self.w_q.shape[0]

    @property
    def d_lr(self) -> int:
        return self.w_q.shape[1]

    def device_wt(self) -> torch.Tensor:
        """[W_q^T ; W_k^T] as one bf16 [2 d_lr, d] device matrix (cached per step)."""
        key = (self.step, id(self.w_q), id(self.w_k))
        if self._dev is None or self._dev[0] != key:
            wt = np.concatenate([self.w_q.T, self.w_k.T], axis=0)
            self._dev = (key, cv.to_device(wt, torch.bfloat16))
        return self._dev[1]


def project(x, w):
    """X W (predictor.py:94-100) on the tcgen05 GEMM: bf16 inputs, fp32 accumulate."""
    x = cv.as_matrix("X", x)
    w = cv.as_matrix("W", w)
    if x.shape[1] != w.shape[0]:
        raise ValueError(f"X has {x.shape[1]} cols but W has {w.shape[0]} rows")
    xd = cv.to_device(x, torch.bfloat16)
    wt = cv.to_device(w.T if not cv.is_torch(w) else w.t(), torch.bfloat16)
    out = ops.gemm_bf16(xd, wt, torch.float32)
    return cv.back(out, x, x.dtype if not cv.is_torch(x) else None)


def estimate_critical(params: PredictorParams, x, k=None, sparsity=None, *, flops=None,
                      return_scores: bool = False) -> CriticalIndexSet:
    """Per-query critical-KV estimate (predictor.py:217-259)."""
    x = cv.as_matrix("X", x)
    s_total = x.shape[0]
    if (k is None) == (sparsity is None):
        raise ValueError("provide exactly one of k or sparsity")
    if sparsity is not None:
        k = k_from_sparsity(sparsity, s_total)
    if x.shape[1] != params.d:
        raise ValueError(f"X has {x.shape[1]} cols but the predictor expects d={params.d}")
    xd = cv.to_device(x, torch.bfloat16)
    lr = ops.gemm_bf16(xd, params.device_wt(), torch.float32)      # [S, 2 d_lr]
    q_lr = lr[:, : params.d_lr].contiguous()
    k_lr = lr[:, params.d_lr:].contiguous()
    if flops is not None:
        flops.projection += 2 * 2 * s_total * params.d * params.d_lr
    if np.ndim(k) == 0:
        k = int(k)
        if not 1 <= k <= s_total:
            raise ValueError(f"k={k} outside [1, {s_total}]")
        res = topk_scores_device(q_lr, k_lr, k, flops=flops, return_scores=return_scores)
        sizes = np.full(s_total, k)
    else:
        sizes = np.asarray(k, dtype=np.int64)
        if sizes.shape != (s_total,):
            raise ValueError(f"per-query k must have shape ({s_total},)")
        if np.any(sizes < 1):
            raise ValueError("per-query k must be >= 1")
        if np.any(sizes > s_total):
            raise ValueError("per-query k exceeds the key count")
        kv = torch.from_numpy(sizes.astype(np.int32)).to(q_lr.device)
        res = topk_scores_device(q_lr, k_lr, kv, flops=flops, return_scores=return_scores)
    idx = res[0].cpu().numpy()
    sets = CriticalIndexSet([idx[i, : sizes[i]] for i in range(s_total)], theta=None)
    return (sets, res[2]) if return_scores else sets
