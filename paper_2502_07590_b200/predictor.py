"""Low-rank critical-KV predictor (reference pkg/src/dynsparse/predictor.py).

Per attention block (the north_star: per head) two projections W_q, W_k in
R^{d x d_lr}; the predicted score matrix (X W_q)(X W_k)^T is ranked per query
and its top-k keys are the critical KV estimate. Here:
  * project            -> host / fp64 inputs: dsv_gemm_f64 (the reference's fp64);
                          bf16 / fp32 torch tensors: K1a tcgen05 GEMM (bf16 in, fp32 acc)
  * estimate_critical  -> the same projection for both sides, then score rows and the
                          exact top-k (fp64 rows + dsv_topk_f64 on the precision path,
                          fp32 rows + K2 otherwise); per-query k arrays use per-row k on
                          the device (same result as the reference's
                          top-k_max + re-rank, predictor.py:246-259, because the
                          top-k set of a row is nested in its top-k_max set).
  * loss_and_grads /   -> the training step (predictor.py:103-214) on
    train_step            device in fp64: Q_lr, K_lr and the final dW contractions are
                          cuBLAS DGEMMs (plain library GEMMs); the [R, S] part — row
                          statistics, G K_lr and G^T Q_lr with G = u_i T + w_i A_hat — are
                          three passes of dsv_pred_pass streaming the target, never
                          materialising A_hat or G. Adam runs on the host copies exactly
                          as the reference (params stay numpy, mutated in place).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _convert as cv
from . import _lib, ops
from .attention import CriticalIndexSet
from .selection import k_from_sparsity, topk_scores_device

COS_WEIGHT = 0.95
NORM_WEIGHT = 0.05
_NORM_FLOOR = 1e-12


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
    """X W (predictor.py:94-100). Host / fp64 inputs: fp64 on the device (dsv_gemm_f64, the
    reference's precision; numpy in -> numpy out in numpy's result dtype). bf16 / fp32 torch
    tensors: the K1a tcgen05 GEMM (bf16 operands, fp32 accumulate)."""
    x = cv.as_matrix("X", x)
    w = cv.as_matrix("W", w)
    if x.shape[1] != w.shape[0]:
        raise ValueError(f"X has {x.shape[1]} cols but W has {w.shape[0]} rows")
    if cv.wants_f64(x) and cv.wants_f64(w):
        out = ops.gemm_f64(cv.to_device(x, torch.float64), cv.to_device(w, torch.float64))
        return cv.back(out, x, cv.result_dtype(x, w))
    xd = cv.to_device(x, torch.bfloat16)
    wt = cv.to_device(w.T if not cv.is_torch(w) else w.t(), torch.bfloat16)
    out = ops.gemm_bf16(xd, wt, torch.float32)
    return cv.back(out, x, x.dtype if not cv.is_torch(x) else None)


def _lowrank(params: PredictorParams, x):
    """(Q_lr, K_lr) on the device: fp64 for host / fp64 inputs (reference precision), else
    the bf16 tcgen05 projection of both sides in one GEMM."""
    if cv.wants_f64(x):
        xd = cv.to_device(x, torch.float64)
        w = torch.from_numpy(np.concatenate([params.w_q, params.w_k], axis=1)).to(xd.device)
        lr = ops.gemm_f64(xd, w)                                         # [S, 2 d_lr] fp64
    else:
        xd = cv.to_device(x, torch.bfloat16)
        lr = ops.gemm_bf16(xd, params.device_wt(), torch.float32)      # [S, 2 d_lr]
    return lr[:, : params.d_lr].contiguous(), lr[:, params.d_lr:].contiguous()


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
    q_lr, k_lr = _lowrank(params, x)
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


def prediction_accuracy(estimated: CriticalIndexSet, oracle: CriticalIndexSet, scores):
    """(recall, score coverage) of an estimate against the oracle sets (predictor.py:262-281):
    mean over queries of |est & oracle| / |oracle| and of mass(est) / mass(oracle) under the
    post-softmax `scores` (1 where the oracle set / mass is empty). The per-query
    intersections and masses are one pass of dsv_set_stats on the device."""
    scores = cv.as_matrix("scores", scores)
    if estimated.n_queries != oracle.n_queries:
        raise ValueError("estimate and oracle cover different query counts")
    n = oracle.n_queries
    if n == 0:
        return float("nan"), float("nan")
    dev = cv.device()
    sc = cv.to_device(scores, torch.float64)
    e_ptr, e_cols = estimated.to_csr(dev)
    o_ptr, o_cols = oracle.to_csr(dev)
    inter, e_mass, o_mass = ops.set_stats_f64(sc, e_ptr, e_cols, o_ptr, o_cols)
    inter = inter.cpu().numpy().astype(np.float64)
    e_mass = e_mass.cpu().numpy()
    o_mass = o_mass.cpu().numpy()
    o_size = oracle.sizes().astype(np.float64)
    recalls = np.where(o_size > 0, inter / np.where(o_size > 0, o_size, 1.0), 1.0)
    cover = np.where(o_mass > 0, e_mass / np.where(o_mass > 0, o_mass, 1.0), 1.0)
    return float(recalls.mean()), float(cover.mean())


def save_checkpoint(params: PredictorParams, directory, block_id: int):
    """predictor.py:284-310: the six matrices as DTSR binary tensors plus canonical JSON
    metadata (serialize.save_tensor format), so reference checkpoints load here and back."""
    from pathlib import Path

    from . import serialize

    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    stem = f"predictor_block{block_id:03d}"
    files = {}
    for tag in ("w_q", "w_k", "m_q", "v_q", "m_k", "v_k"):
        path = directory / f"{stem}.{tag}.bin"
        serialize.save_tensor(path, getattr(params, tag))
        files[tag] = path.name
    meta = {"block_id": block_id, "d": params.d, "d_lr": params.d_lr, "lr": params.lr,
            "step": params.step, "loss_history": params.loss_history, "files": files}
    meta_path = directory / f"{stem}.json"
    meta_path.write_text(serialize.canonical_json(meta))
    return meta_path


def load_checkpoint(meta_path) -> PredictorParams:
    """predictor.py:313-324."""
    import json
    from pathlib import Path

    from . import serialize

    meta_path = Path(meta_path)
    meta = json.loads(meta_path.read_text())
    arr = {tag: serialize.load_tensor(meta_path.parent / name) for tag, name in meta["files"].items()}
    return PredictorParams(w_q=arr["w_q"], w_k=arr["w_k"], lr=meta["lr"], step=meta["step"],
                           m_q=arr["m_q"], v_q=arr["v_q"], m_k=arr["m_k"], v_k=arr["v_k"],
                           loss_history=list(meta["loss_history"]))


@dataclass
class PredictorLossReport:
    """predictor.py:86-91."""

    cos_loss: float
    norm_loss: float
    total: float
    step_skipped: bool = False


def predictor_loss(a_hat, a_target) -> PredictorLossReport:
    """Composite loss between given predicted and true score rows (predictor.py:139-148)."""
    a_hat = np.asarray(cv.as_matrix("A_hat", a_hat), dtype=np.float64)
    a_target = np.asarray(cv.as_matrix("A_target", a_target), dtype=np.float64)
    if a_hat.shape != a_target.shape:
        raise ValueError(f"shape mismatch: {a_hat.shape} vs {a_target.shape}")
    n = a_hat.shape[0]
    an, tn = np.linalg.norm(a_hat, axis=1), np.linalg.norm(a_target, axis=1)
    live = tn > _NORM_FLOOR
    nz = live & (an > _NORM_FLOOR)
    cos = np.zeros(n)
    cos[nz] = np.sum(a_hat[nz] * a_target[nz], axis=1) / (an[nz] * tn[nz])
    cos_loss = float(np.sum(np.where(live, 1.0 - cos, 0.0)) / n)
    norm_loss = float(np.linalg.norm(a_hat - a_target)) / max(float(np.linalg.norm(a_target)), _NORM_FLOOR)
    return PredictorLossReport(cos_loss, norm_loss, COS_WEIGHT * cos_loss + NORM_WEIGHT * norm_loss)


def _dev_f64(t, dev):
    if isinstance(t, torch.Tensor):
        return t.to(device=dev, dtype=torch.float64)
    return torch.as_tensor(np.asarray(t, dtype=np.float64), device=dev)


def loss_and_grads(params: PredictorParams, x, a_target, rows=None, device="cuda"):
    """Loss report plus analytic gradients w.r.t. W_q and W_k (predictor.py:151-194).

    x [S, d]; a_target [R, S] (R = len(rows) or S), numpy or device tensor (fp32 / fp64).
    Returns (PredictorLossReport, grad_wq, grad_wk) with numpy fp64 gradients.
    """
    dev = torch.device(device)
    xm = cv.as_matrix("X", x)
    if xm.shape[1] != params.d:
        raise ValueError(f"X has {xm.shape[1]} cols but W_q has {params.d} rows")
    X = _dev_f64(xm, dev)
    Xr = X if rows is None else X.index_select(0, torch.as_tensor(np.asarray(rows, dtype=np.int64), device=dev))
    R, S = Xr.shape[0], X.shape[0]
    if isinstance(a_target, torch.Tensor):
        T = a_target.to(dev)
        if T.dtype not in (torch.float32, torch.float64):
            T = T.double()
    else:
        T = torch.as_tensor(np.asarray(a_target, dtype=np.float64), device=dev)
    if T.dim() != 2 or tuple(T.shape) != (R, S):
        raise ValueError(f"A_target must be ({R}, {S}), got {tuple(T.shape)}")
    T = T.contiguous()
    wq, wk = _dev_f64(params.w_q, dev), _dev_f64(params.w_k, dev)
    q_lr = (Xr @ wq).contiguous()                       # [R, r]
    k_lr = (X @ wk).contiguous()                        # [S, r]
    r = q_lr.shape[1]
    tdt = _lib.DTYPE_F64 if T.dtype == torch.float64 else _lib.DTYPE_F32
    stats = torch.empty((R, 4), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("dsv_pred_pass", 0, q_lr.data_ptr(), k_lr.data_ptr(), T.data_ptr(), tdt, T.stride(0),
              R, S, r, 0, stats.data_ptr(), st)
    a2, t2, at, d2 = stats.unbind(1)
    an, tn = a2.sqrt(), t2.sqrt()
    live = tn > _NORM_FLOOR
    nz = live & (an > _NORM_FLOOR)
    one = torch.ones_like(an)
    cos = torch.where(nz, at / torch.where(nz, an * tn, one), torch.zeros_like(an))
    cos_loss = float(torch.where(live, 1.0 - cos, torch.zeros_like(cos)).sum().item()) / R
    denom = max(float(t2.sum().sqrt().item()), _NORM_FLOOR)
    dist = float(d2.sum().sqrt().item())
    # G[i, :] = u_i T[i, :] + w_i A_hat[i, :]
    u = torch.where(nz, -1.0 / (torch.where(nz, an * tn, one) * R), torch.zeros_like(an)) * COS_WEIGHT
    w = torch.where(nz, cos / (torch.where(nz, an * an, one) * R), torch.zeros_like(an)) * COS_WEIGHT
    if dist > _NORM_FLOOR:
        u = u - NORM_WEIGHT / (denom * dist)
        w = w + NORM_WEIGHT / (denom * dist)
    uw = torch.stack([u, w], dim=1).contiguous()
    g1 = torch.empty((R, r), dtype=torch.float64, device=dev)
    g2 = torch.empty((S, r), dtype=torch.float64, device=dev)
    _lib.call("dsv_pred_pass", 1, q_lr.data_ptr(), k_lr.data_ptr(), T.data_ptr(), tdt, T.stride(0),
              R, S, r, uw.data_ptr(), g1.data_ptr(), st)
    _lib.call("dsv_pred_pass", 2, q_lr.data_ptr(), k_lr.data_ptr(), T.data_ptr(), tdt, T.stride(0),
              R, S, r, uw.data_ptr(), g2.data_ptr(), st)
    grad_wq = (Xr.t() @ g1).cpu().numpy()
    grad_wk = (X.t() @ g2).cpu().numpy()
    norm_loss = dist / denom
    report = PredictorLossReport(cos_loss, norm_loss, COS_WEIGHT * cos_loss + NORM_WEIGHT * norm_loss)
    return report, grad_wq, grad_wk


def _adam_update(w, grad, m, v, lr, beta1, beta2, eps, step):
    """predictor.py:197-204 (host, in place)."""
    m *= beta1
    m += (1.0 - beta1) * grad
    v *= beta2
    v += (1.0 - beta2) * grad**2
    w -= lr * (m / (1.0 - beta1**step)) / (np.sqrt(v / (1.0 - beta2**step)) + eps)


def train_step(params: PredictorParams, x, a_target, rows=None, device="cuda") -> PredictorLossReport:
    """One Adam step on the device gradients; mutates `params` (predictor.py:207-214).
    A non-finite gradient skips the update and flags the report."""
    report, gq, gk = loss_and_grads(params, x, a_target, rows=rows, device=device)
    if not (np.all(np.isfinite(gq)) and np.all(np.isfinite(gk))):
        report.step_skipped = True
        params.loss_history.append(report.total)
        return report
    params.step += 1
    _adam_update(params.w_q, gq, params.m_q, params.v_q, params.lr, params.beta1, params.beta2,
                 params.eps, params.step)
    _adam_update(params.w_k, gk, params.m_k, params.v_k, params.lr, params.beta1, params.beta2,
                 params.eps, params.step)
    params.loss_history.append(report.total)
    return report
