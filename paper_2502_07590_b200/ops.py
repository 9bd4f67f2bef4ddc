"""Device-tensor wrappers over the C ABI (one function per libdsv entry point).

All tensors must already live on the current CUDA device; outputs are
allocated here with torch (device memory plumbing only) and filled by the
libdsv kernels on the current stream. There is no CPU path: a missing CUDA
device or library raises.
"""

from __future__ import annotations

import math

import torch

from . import _lib

_F32, _BF16 = _lib.DTYPE_F32, _lib.DTYPE_BF16


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _require_cuda(*ts) -> None:
    cur = None
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise _lib.DSVError("libdsv kernels need CUDA tensors (no CPU fallback exists)")
        if cur is None:
            cur = torch.cuda.current_device()
        if t.device.index != cur:
            # the C ABI launches on the calling thread's current device and stream
            raise _lib.DSVError(f"tensor on {t.device} while the current device is cuda:{cur}; "
                                "call under torch.cuda.device(tensor.device)")


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


# ------------------------------------------------------------------- K1 GEMM
def gemm_bf16(a: torch.Tensor, b: torch.Tensor, out_dtype=torch.float32, out=None) -> torch.Tensor:
    """Batched C = A . B^T on tcgen05. a: [nb, M, K] or [M, K] bf16, b: [nb, N, K] or [N, K].

    out: optional preallocated C (unit stride along N) of the result's shape and dtype.
    """
    _require_cuda(a, b)
    squeeze = a.dim() == 2
    if squeeze:
        a, b = a.unsqueeze(0), b.unsqueeze(0)
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise ValueError("gemm_bf16 expects bf16 operands")
    nb, M, K = a.shape
    _, N, K2 = b.shape
    if K != K2 or b.shape[0] != nb:
        raise ValueError(f"gemm shape mismatch {tuple(a.shape)} x {tuple(b.shape)}")
    if a.stride(2) != 1 or b.stride(2) != 1:
        raise ValueError("gemm operands need unit stride along K")
    if out is None:
        c = torch.empty((nb, M, N), device=a.device, dtype=out_dtype)
    else:
        c = out.unsqueeze(0) if squeeze else out
        if tuple(c.shape) != (nb, M, N) or c.dtype != out_dtype or c.stride(2) != 1:
            raise ValueError("gemm out has the wrong shape, dtype or layout")
    _lib.call("dsv_gemm_bf16", _ptr(a), a.stride(1), a.stride(0), _ptr(b), b.stride(1), b.stride(0),
              _ptr(c), _F32 if out_dtype == torch.float32 else _BF16, c.stride(1), c.stride(0),
              M, N, K, nb, _stream())
    return c[0] if squeeze else c


def project(x: torch.Tensor, wt: torch.Tensor) -> torch.Tensor:
    """K1a: [L, d_model] . wt[n_out, d_model]^T -> [L, n_out] bf16."""
    _require_cuda(x, wt)
    x = x.contiguous()
    wt = wt.contiguous()
    L, dm = x.shape
    n_out = wt.shape[0]
    out = torch.empty((L, n_out), device=x.device, dtype=torch.bfloat16)
    _lib.call("dsv_project", _ptr(x), _ptr(wt), _ptr(out), L, dm, n_out, _stream())
    return out


def scores_f32(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """fp32 scores C[nb, R, Lk] = A[nb, R, r] . B[nb, Lk, r]^T (A, B fp32 or bf16)."""
    _require_cuda(a, b)
    squeeze = a.dim() == 2
    if squeeze:
        a, b = a.unsqueeze(0), b.unsqueeze(0)
    if a.dtype != b.dtype or a.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("scores_f32 expects matching fp32 or bf16 operands")
    if a.stride(2) != 1 or b.stride(2) != 1:
        a, b = a.contiguous(), b.contiguous()
    nb, R, r = a.shape
    Lk = b.shape[1]
    if out is None:
        out = torch.empty((nb, R, Lk), device=a.device, dtype=torch.float32)
    _lib.call("dsv_scores_f32", _ptr(a), a.stride(1), a.stride(0), _ptr(b), b.stride(1),
              b.stride(0), _ptr(out), out.stride(1), out.stride(0), nb, R, Lk, r,
              _BF16 if a.dtype == torch.bfloat16 else _F32, _stream())
    return out[0] if squeeze else out


def proxy_scores(qp: torch.Tensor, k_lr: torch.Tensor, out: torch.Tensor | None = None):
    """K1b on tcgen05: [H, G, r] . [H, L, r]^T -> fp32 [H, G, L] (r = 16, strided views ok)."""
    _require_cuda(qp, k_lr)
    H, G, r = qp.shape
    L = k_lr.shape[1]
    if qp.stride(2) != 1 or k_lr.stride(2) != 1:
        raise ValueError("proxy_scores operands need unit stride along r")
    if out is None:
        out = torch.empty((H, G, L), device=qp.device, dtype=torch.float32)
    _lib.call("dsv_proxy_scores", _ptr(qp), qp.stride(1), qp.stride(0), _ptr(k_lr), k_lr.stride(1),
              k_lr.stride(0), _ptr(out), out.stride(1), out.stride(0), H, G, L, r, _stream())
    return out


# ------------------------------------------------------------------- K2 top-k
def topk_rows(scores: torch.Tensor, k_per_head: torch.Tensor, rows_per_head: int,
              k_max: int | None = None, out=None):
    """Exact top-k per row of fp32 scores [R, L] (row r uses k_per_head[r // rows_per_head]).

    Returns (idx int32 [R, k_max] ascending — entries past a row's k are
    undefined, thresholds fp32 [R]). out: optional preallocated (idx, thr) pair.
    """
    _require_cuda(scores, k_per_head)
    if scores.dtype != torch.float32 or scores.dim() != 2 or scores.stride(1) != 1:
        raise ValueError("scores must be a row-major fp32 matrix")
    R, L = scores.shape
    kp = k_per_head.to(device=scores.device, dtype=torch.int32).contiguous()
    if k_max is None:
        k_max = int(kp.max().item())
    if out is None:
        idx = torch.empty((R, k_max), device=scores.device, dtype=torch.int32)
        thr = torch.empty((R,), device=scores.device, dtype=torch.float32)
    else:
        idx, thr = out
        if (idx.dtype != torch.int32 or idx.shape[0] != R or idx.shape[1] < k_max or idx.stride(1) != 1
                or thr.dtype != torch.float32 or thr.shape != (R,) or not thr.is_contiguous()):
            raise ValueError("topk out must be (int32 [R, >=k_max] rows, fp32 [R])")
    _lib.call("dsv_topk", _ptr(scores), scores.stride(0), R, L, _ptr(kp), rows_per_head, _ptr(idx),
              idx.stride(0), _ptr(thr), _stream())
    return idx, thr


_WS_CACHE = {}


def select_workspace(H: int, G: int, L: int, k_max: int, split: int, device) -> torch.Tensor | None:
    """Device workspace of the single-pass fused selection (cached per shape / device); None
    where the library advises the multi-pass algorithm."""
    key = (H, G, L, k_max, split, str(device))
    if key not in _WS_CACHE and len(_WS_CACHE) >= 8:     # bounded: a few live shapes at most
        _WS_CACHE.pop(next(iter(_WS_CACHE)))
    if key not in _WS_CACHE:
        n = int(_lib.load().dsv_select_fused_workspace_size(H, G, L, k_max, split))
        _WS_CACHE[key] = torch.empty((n,), dtype=torch.uint8, device=device) if n > 0 else None
    return _WS_CACHE[key]


def select_fast_fallbacks(H: int, G: int, L: int, k_max: int, split: int, device) -> int:
    """Row tiles the last single-pass selection of this shape re-ran with the multi-pass
    algorithm (the workspace's leading tile-flag array; diagnostics). -1: no workspace."""
    ws = _WS_CACHE.get((H, G, L, k_max, split, str(device)))
    if ws is None:
        return -1
    n_mt = H * ((G + 127) // 128)
    return int(ws[: 4 * n_mt].view(torch.int32).ne(0).sum().item())


def select_band_stats(H: int, G: int, L: int, k_max: int, split: int, S: int, device):
    """(mean, max) band entries per (row, CTA) of the last single-pass selection of this shape
    (the workspace's count array; diagnostics for the band sizing)."""
    ws = _WS_CACHE.get((H, G, L, k_max, split, str(device)))
    if ws is None:
        return None
    n_mt = H * ((G + 127) // 128)
    off = (n_mt * 4 + 255) // 256 * 256
    c = ws[off: off + 4 * H * G * S].view(torch.int32).double()
    return float(c.mean().item()), int(c.max().item())


def select_fused(q_prox: torch.Tensor, k_lr: torch.Tensor, k_per_head: torch.Tensor,
                 k_max: int | None = None, split: int = 0, out=None, mode: str = "auto"):
    """K1b + K2 fused (select_fused.cu): exact top-k of q_prox[h] . k_lr[h]^T per row.

    q_prox [H, G, r], k_lr [H, L, r] bf16 with unit stride along r (r <= 16). Same result as
    topk_rows(gemm_bf16(q_prox, k_lr), k_per_head, G) without the [H, G, L] fp32 scores.
    Returns (idx int32 [H*G, k_max], thr fp32 [H*G]); out: optional preallocated pair.
    mode: "fast" (single collect pass + finish, a cached workspace), "multipass" (no
    workspace), "auto" = fast unless DSV_SELECT_MULTIPASS=1. Results are identical.
    """
    _require_cuda(q_prox, k_lr, k_per_head)
    if q_prox.dtype != torch.bfloat16 or k_lr.dtype != torch.bfloat16:
        raise ValueError("select_fused expects bf16 operands")
    if q_prox.dim() != 3 or k_lr.dim() != 3 or q_prox.stride(2) != 1 or k_lr.stride(2) != 1:
        raise ValueError("select_fused operands must be [H, rows, r] with unit stride along r")
    H, G, r = q_prox.shape
    H2, L, r2 = k_lr.shape
    if H2 != H or r2 != r:
        raise ValueError(f"select_fused shape mismatch {tuple(q_prox.shape)} x {tuple(k_lr.shape)}")
    kp = k_per_head.to(device=q_prox.device, dtype=torch.int32).contiguous()
    if k_max is None:
        k_max = int(kp.max().item())
    if out is None:
        idx = torch.empty((H * G, k_max), device=q_prox.device, dtype=torch.int32)
        thr = torch.empty((H * G,), device=q_prox.device, dtype=torch.float32)
    else:
        idx, thr = out
    if mode == "auto":
        import os

        mode = "multipass" if os.environ.get("DSV_SELECT_MULTIPASS") == "1" else "fast"
    ws = select_workspace(H, G, L, int(k_max), int(split), q_prox.device) if mode == "fast" else None
    _lib.call("dsv_select_fused", _ptr(q_prox), q_prox.stride(1), q_prox.stride(0), _ptr(k_lr),
              k_lr.stride(1), k_lr.stride(0), H, G, L, r, _ptr(kp), _ptr(idx), idx.stride(0),
              _ptr(thr), int(split), _ptr(ws), 0 if ws is None else ws.numel(), _stream())
    return idx, thr


# ------------------------------------------------------------------- K3 attention
def sparse_fwd(q, k, v, grp_rows, grp_size, idx, kcount, scale=None, kcount_hg=None, zero=None,
               tile_grp=None, out_rows=None):
    """Group-tiled sparse attention forward. q: [H, Lq, D], k/v: [H, Lk, D] bf16.

    grp_rows int32 [G, 128], grp_size int32 [G], idx int32 [H, G, ldk], kcount int32 [H]
    (or per-row counts kcount_hg int32 [H, G]). Returns (out bf16 [H, Lq, D], lse2 fp32 [H, Lq]).
    zero: optional contiguous fp32 tensor the kernel sets to 0 while it runs (the backward's
    dK/dV accumulators).
    tile_grp: optional int32 [G] tile -> voxel group map (groups of more than 128 queries span
    several tiles that share the group's idx row; idx / kcount_hg are then per group).
    out_rows: optional (tab int64 [H * n], n, chunk): output rows are also stored at the token
    owners' addresses (fused HCP output redistribution).
    """
    _require_cuda(q, k, v, grp_rows, grp_size, idx, kcount)
    if zero is not None and (zero.dtype != torch.float32 or not zero.is_contiguous()):
        raise ValueError("sparse_fwd: zero must be a contiguous fp32 tensor")
    H, Lq, D = q.shape
    Lk = k.shape[1]
    G = grp_rows.shape[0]
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    out = torch.empty_like(q)
    lse = torch.empty((H, Lq), device=q.device, dtype=torch.float32)
    work = torch.empty((H * G + 2,), device=q.device, dtype=torch.int32)
    _lib.call("dsv_sparse_fwd", _ptr(q), _ptr(k), _ptr(v), _ptr(grp_rows), _ptr(grp_size),
              _ptr(idx), idx.stride(1), _ptr(kcount), _ptr(kcount_hg), H, G, Lq, Lk, D,
              float(scale), _ptr(out), _ptr(lse), _ptr(work), work.numel(), _ptr(zero),
              0 if zero is None else zero.numel(), _ptr(tile_grp),
              0 if tile_grp is None else idx.shape[1], *_rows_args(out_rows), _stream())
    return out, lse


def _rows_args(rows):
    if rows is None:
        return 0, 0, 0
    tab, n, chunk = rows
    if tab.dtype != torch.int64 or not tab.is_cuda:
        raise ValueError("row table must be an int64 CUDA tensor")
    return tab.data_ptr(), int(n), int(chunk)


def sparse_bwd(q, k, v, out, dout, lse, grp_rows, grp_size, idx, kcount, scale=None,
               dk_acc=None, dv_acc=None, kcount_hg=None, tile_grp=None, dq_rows=None,
               dkdv_out=None, dkdv_rows=None):
    """Backward of sparse_fwd. Returns (dq bf16, dk_acc fp32, dv_acc fp32).

    dkdv_out (bf16 [2, H, Lk, D]) or dkdv_rows ((tab, n, chunk) for dK and for dV): the
    kernel also converts the accumulators to bf16 there in its tail
    (dsv_sparse_bwd_convert)."""
    _require_cuda(q, k, v, out, dout, lse)
    H, Lq, D = q.shape
    Lk = k.shape[1]
    G = grp_rows.shape[0]
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    dq = torch.empty_like(q)
    if dk_acc is None:
        dk_acc = torch.zeros((H, Lk, D), device=q.device, dtype=torch.float32)
    if dv_acc is None:
        dv_acc = torch.zeros((H, Lk, D), device=q.device, dtype=torch.float32)
    work = torch.empty((4,), device=q.device, dtype=torch.int32)
    if dkdv_out is None and dkdv_rows is None:
        _lib.call("dsv_sparse_bwd", _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(dout), _ptr(lse),
                  _ptr(grp_rows), _ptr(grp_size), _ptr(idx), idx.stride(1), _ptr(kcount),
                  _ptr(kcount_hg), H, G, Lq, Lk, D, float(scale), _ptr(dq), _ptr(dk_acc),
                  _ptr(dv_acc), _ptr(work), _ptr(tile_grp), 0 if tile_grp is None else idx.shape[1],
                  *_rows_args(dq_rows), _stream())
        return dq, dk_acc, dv_acc
    if dkdv_out is not None:
        _require_cuda(dkdv_out)
        if (dkdv_out.dtype != torch.bfloat16 or dkdv_out.shape != (2, H, Lk, D)
                or not dkdv_out.is_contiguous()):
            raise ValueError("sparse_bwd: dkdv_out must be a contiguous bf16 [2, H, Lk, D] tensor")
        ktab, vtab, kv_n, kv_chunk = 0, 0, 0, 0
    else:
        ktab, kv_n, kv_chunk = _rows_args(dkdv_rows[0])
        vtab = _rows_args(dkdv_rows[1])[0]
    conv = torch.empty((H + 1,), device=q.device, dtype=torch.int32)
    _lib.call("dsv_sparse_bwd_convert", _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(dout),
              _ptr(lse), _ptr(grp_rows), _ptr(grp_size), _ptr(idx), idx.stride(1), _ptr(kcount),
              _ptr(kcount_hg), H, G, Lq, Lk, D, float(scale), _ptr(dq), _ptr(dk_acc),
              _ptr(dv_acc), _ptr(work), _ptr(tile_grp), 0 if tile_grp is None else idx.shape[1],
              *_rows_args(dq_rows), _ptr(dkdv_out), ktab, vtab, kv_n, kv_chunk, _ptr(conv),
              _stream())
    return dq, dk_acc, dv_acc


def rows_fwd(q, k, v, ptr, cols, scale=None):
    """Ragged CSR sparse attention forward on CUDA cores (cols None = every key).

    Returns (out fp32, lse fp32 natural)."""
    _require_cuda(q, k, v, ptr, cols)
    H, Lq, D = q.shape
    Lk = k.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    out = torch.empty((H, Lq, D), device=q.device, dtype=torch.float32)
    lse = torch.empty((H, Lq), device=q.device, dtype=torch.float32)
    _lib.call("dsv_rows_fwd", _ptr(q), _ptr(k), _ptr(v), _ptr(ptr), _ptr(cols), H, Lq, Lk, D,
              float(scale), _BF16 if q.dtype == torch.bfloat16 else _F32, _ptr(out), _ptr(lse),
              _stream())
    return out, lse


def rows_bwd(q, k, v, out, lse, dout, ptr, cols, scale=None):
    """Backward of rows_fwd. Returns fp32 (dq, dk, dv)."""
    _require_cuda(q, k, v, out, lse, dout, ptr, cols)
    H, Lq, D = q.shape
    Lk = k.shape[1]
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    dq = torch.empty((H, Lq, D), device=q.device, dtype=torch.float32)
    dk = torch.zeros((H, Lk, D), device=q.device, dtype=torch.float32)
    dv = torch.zeros((H, Lk, D), device=q.device, dtype=torch.float32)
    _lib.call("dsv_rows_bwd", _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(dout),
              _ptr(ptr), _ptr(cols), H, Lq, Lk, D, float(scale),
              _BF16 if q.dtype == torch.bfloat16 else _F32, _ptr(dq), _ptr(dk), _ptr(dv),
              _stream())
    return dq, dk, dv


def gather_rows(src: torch.Tensor, rows: torch.Tensor, out: torch.Tensor | None = None):
    """out[i] = src[rows[i]] for a 2-D src (row-major rows)."""
    _require_cuda(src, rows)
    rows = rows.to(torch.int32).contiguous()
    n = rows.numel()
    if src.dim() != 2 or src.stride(1) != 1:
        raise ValueError("gather_rows: src must be 2-D with unit column stride")
    if out is not None and (out.dim() != 2 or out.stride(1) != 1 or out.shape[0] != n
                            or out.shape[1] != src.shape[1] or out.dtype != src.dtype):
        raise ValueError("gather_rows: out must be [len(rows), src.shape[1]] with unit column stride")
    if out is None:
        out = torch.empty((n, src.shape[1]), device=src.device, dtype=src.dtype)
    es = src.element_size()
    _lib.call("dsv_gather_rows", _ptr(src), src.stride(0) * es, _ptr(rows), n, src.shape[1] * es,
              _ptr(out), out.stride(0) * es, _stream())
    return out


def critical_counts(scores: torch.Tensor, sqrt_d: float, theta: float) -> torch.Tensor:
    """Critical-KV prefix length per row of raw fp32 scores [R, L] (dsv_critical_counts)."""
    _require_cuda(scores)
    if scores.dtype != torch.float32 or scores.dim() != 2 or scores.stride(1) != 1:
        raise ValueError("critical_counts: scores must be a row-major fp32 matrix")
    out = torch.empty((scores.shape[0],), dtype=torch.int32, device=scores.device)
    _lib.call("dsv_critical_counts", _ptr(scores), scores.stride(0), scores.shape[0], scores.shape[1],
              float(sqrt_d), float(theta), _ptr(out), _stream())
    return out


def copy_jobs(jobs: torch.Tensor, splits: int = 16, threads: int = 256) -> None:
    """Run a [njobs, 6] int64 device job table (src, dst, src_stride, dst_stride, rows,
    row_bytes) in one launch (dsv_copy_jobs); addresses may be NVLink peer pointers.
    threads = 128: blocks small enough to share an SM with a persistent attention CTA."""
    _require_cuda(jobs)
    if jobs.dtype != torch.int64 or jobs.dim() != 2 or jobs.shape[1] != 6 or not jobs.is_contiguous():
        raise ValueError("copy_jobs: expected a contiguous [njobs, 6] int64 table")
    if threads == 256:
        _lib.call("dsv_copy_jobs", _ptr(jobs), jobs.shape[0], int(splits), _stream())
    else:
        _lib.call("dsv_copy_jobs_threads", _ptr(jobs), jobs.shape[0], int(splits), int(threads),
                  _stream())


def f32_to_bf16_rows(x: torch.Tensor, rows) -> None:
    """fp32 [H, L, D] -> bf16 rows at the (tab, n, chunk) addresses (dsv_f32_to_bf16_rows)."""
    _require_cuda(x)
    if x.dtype != torch.float32 or x.dim() != 3 or not x.is_contiguous():
        raise ValueError("f32_to_bf16_rows expects a contiguous fp32 [H, L, D] tensor")
    tab, n, chunk = _rows_args(rows)
    _lib.call("dsv_f32_to_bf16_rows", _ptr(x), x.shape[0], x.shape[1], x.shape[2], tab, n, chunk,
              _stream())


def f32_to_bf16(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    _require_cuda(x)
    x = x.contiguous()
    if out is None:
        out = torch.empty(x.shape, device=x.device, dtype=torch.bfloat16)
    _lib.call("dsv_f32_to_bf16", _ptr(x), _ptr(out), x.numel(), _stream())
    return out


# ------------------------------------------------------------------- ring KV pass
def _contig(*ts):
    for t in ts:
        if t is not None and not t.is_contiguous():
            raise ValueError("ring kernels need contiguous tensors")


def ring_lse_merge(acc, lse_in, lse_out, part, lse_part, first: bool, out=None) -> None:
    """acc fp32 [..., D] / lse_in -> lse_out fp32 [...]: merge one hop's partial (part bf16,
    lse_part log2 domain). first: acc := part. out (bf16, optional): the merged rows."""
    _require_cuda(acc, part, lse_part, lse_out)
    _contig(acc, lse_in, lse_out, part, lse_part, out)
    D = acc.shape[-1]
    rows = acc.numel() // D
    if part.shape != acc.shape or lse_part.numel() != rows or lse_out.numel() != rows:
        raise ValueError("ring_lse_merge: shape mismatch")
    _lib.call("dsv_ring_lse_merge", _ptr(acc), _ptr(lse_in), _ptr(lse_out), _ptr(part),
              _ptr(lse_part), rows, D, int(first), _ptr(out), _stream())


def ring_accum_bf16(acc, x, first: bool, out=None) -> None:
    """acc fp32 := (first ? 0 : acc) + x (bf16); out (bf16, optional) = the sum."""
    _require_cuda(acc, x)
    _contig(acc, x, out)
    if x.numel() != acc.numel():
        raise ValueError("ring_accum_bf16: shape mismatch")
    _lib.call("dsv_ring_accum_bf16", _ptr(acc), _ptr(x), acc.numel(), int(first), _ptr(out), _stream())


def ring_accum_f32(acc, part, first: bool) -> None:
    """acc := (first ? 0 : acc) + part; part := 0."""
    _require_cuda(acc, part)
    _contig(acc, part)
    if part.numel() != acc.numel():
        raise ValueError("ring_accum_f32: shape mismatch")
    _lib.call("dsv_ring_accum_f32", _ptr(acc), _ptr(part), acc.numel(), int(first), _stream())


# ------------------------------------------------------------------- fp64 precision path
_F64 = torch.float64


def _need_f64(*ts):
    for t in ts:
        if t is not None and t.dtype != _F64:
            raise ValueError("fp64 kernels need float64 tensors")


def gemm_f64(a: torch.Tensor, b: torch.Tensor, div: float = 1.0, out=None) -> torch.Tensor:
    """fp64 C = (A . B) / div on CUDA cores (dsv_gemm_f64). a: [M, K] or [nb, M, K],
    b: [K, N] or [nb, K, N]; any strides (pass b = x.t() for A . x^T)."""
    _require_cuda(a, b)
    _need_f64(a, b)
    squeeze = a.dim() == 2
    if squeeze:
        a, b = a.unsqueeze(0), b.unsqueeze(0)
    nb, M, K = a.shape
    if b.shape[0] != nb or b.shape[1] != K:
        raise ValueError(f"gemm_f64 shape mismatch {tuple(a.shape)} x {tuple(b.shape)}")
    N = b.shape[2]
    if out is None:
        c = torch.empty((nb, M, N), device=a.device, dtype=_F64)
    else:
        c = out.unsqueeze(0) if squeeze else out
        if tuple(c.shape) != (nb, M, N) or c.dtype != _F64 or c.stride(2) != 1:
            raise ValueError("gemm_f64 out has the wrong shape, dtype or layout")
    _lib.call("dsv_gemm_f64", _ptr(a), a.stride(1), a.stride(2), a.stride(0), _ptr(b), b.stride(1),
              b.stride(2), b.stride(0), _ptr(c), c.stride(1), c.stride(0), M, N, K, nb, float(div),
              _stream())
    return c[0] if squeeze else c


def softmax_rows_f64_(x: torch.Tensor) -> torch.Tensor:
    """In place: every row of the fp64 matrix x becomes its max-subtracted softmax."""
    _require_cuda(x)
    _need_f64(x)
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("softmax_rows_f64_ expects a row-major fp64 matrix")
    _lib.call("dsv_softmax_rows_f64", _ptr(x), x.stride(0), x.shape[0], x.shape[1], _stream())
    return x


def topk_f64(scores: torch.Tensor, k_per, rows_per_k: int, k_max: int):
    """Exact top-k per row of fp64 scores [R, L] (dsv_topk_f64). k_per: int32 device tensor,
    row r uses k_per[r // rows_per_k]. Returns (idx int32 [R, k_max], thr fp64 [R])."""
    _require_cuda(scores, k_per)
    _need_f64(scores)
    if scores.dim() != 2 or scores.stride(1) != 1:
        raise ValueError("topk_f64 expects a row-major fp64 matrix")
    R, L = scores.shape
    kp = k_per.to(device=scores.device, dtype=torch.int32).contiguous()
    idx = torch.empty((R, k_max), device=scores.device, dtype=torch.int32)
    thr = torch.empty((R,), device=scores.device, dtype=_F64)
    _lib.call("dsv_topk_f64", _ptr(scores), scores.stride(0), R, L, _ptr(kp), int(rows_per_k),
              _ptr(idx), idx.stride(0), _ptr(thr), _stream())
    return idx, thr


def rows_fwd_f64(q, k, v, ptr, cols, scale):
    """fp64 attention over CSR lists (cols None: every key). q [H, Lq, Dk], k [H, Lk, Dk],
    v [H, Lk, Dv] -> (out [H, Lq, Dv], lse [H, Lq]) fp64."""
    _require_cuda(q, k, v)
    _need_f64(q, k, v)
    H, Lq, Dk = q.shape
    Lk, Dv = k.shape[1], v.shape[2]
    out = torch.empty((H, Lq, Dv), device=q.device, dtype=_F64)
    lse = torch.empty((H, Lq), device=q.device, dtype=_F64)
    _lib.call("dsv_rows_fwd_f64", _ptr(q), _ptr(k), _ptr(v), _ptr(ptr), _ptr(cols), H, Lq, Lk, Dk,
              Dv, float(scale), _ptr(out), _ptr(lse), _stream())
    return out, lse


def rows_bwd_f64(q, k, v, out, lse, dout, ptr, cols, scale):
    """Backward of rows_fwd_f64 -> fp64 (dq, dk, dv)."""
    _require_cuda(q, k, v, out, lse, dout)
    _need_f64(q, k, v, out, lse, dout)
    H, Lq, Dk = q.shape
    Lk, Dv = k.shape[1], v.shape[2]
    dq = torch.empty_like(q)
    dk = torch.zeros((H, Lk, Dk), device=q.device, dtype=_F64)
    dv = torch.zeros((H, Lk, Dv), device=q.device, dtype=_F64)
    _lib.call("dsv_rows_bwd_f64", _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(dout),
              _ptr(ptr), _ptr(cols), H, Lq, Lk, Dk, Dv, float(scale), _ptr(dq), _ptr(dk), _ptr(dv),
              _stream())
    return dq, dk, dv


def sorted_stats_f64(scores: torch.Tensor, theta: float = 0.0, eps: float = 0.0, top_n: int = 0,
                     want_keep: bool = True, want_top: bool = False):
    """Per row of non-negative fp64 scores: (n_keep int32 [R] | None, topmass fp64 [R] | None)
    (dsv_sorted_stats_f64: the critical-prefix length and the top-n mass of the sorted row)."""
    _require_cuda(scores)
    _need_f64(scores)
    if scores.dim() != 2 or scores.stride(1) != 1:
        raise ValueError("sorted_stats_f64 expects a row-major fp64 matrix")
    R, L = scores.shape
    keep = torch.empty((R,), device=scores.device, dtype=torch.int32) if want_keep else None
    top = torch.empty((R,), device=scores.device, dtype=_F64) if want_top else None
    nbytes = int(load_lib().dsv_sorted_stats_scratch_bytes(R, L))
    scratch = torch.empty((max(nbytes, 1),), device=scores.device, dtype=torch.uint8) if nbytes else None
    _lib.call("dsv_sorted_stats_f64", _ptr(scores), scores.stride(0), R, L, float(theta), float(eps),
              int(top_n), _ptr(keep), _ptr(top), _ptr(scratch), nbytes, _stream())
    return keep, top


def histogram_f64(values: torch.Tensor, edges: torch.Tensor) -> torch.Tensor:
    """np.histogram(values, bins=edges) counts on the device (int64 [len(edges) - 1])."""
    _require_cuda(values, edges)
    _need_f64(values, edges)
    v = values if values.dim() == 2 else values.reshape(1, -1)
    if v.stride(-1) != 1:
        v = v.contiguous()
    nb = edges.numel() - 1
    counts = torch.zeros((nb,), device=values.device, dtype=torch.int64)
    _lib.call("dsv_histogram_f64", _ptr(v), v.stride(0), v.shape[0], v.shape[1],
              _ptr(edges.contiguous()), nb, _ptr(counts), _stream())
    return counts


def load_lib():
    return _lib.load()


def set_stats_f64(scores: torch.Tensor, e_ptr, e_cols, o_ptr, o_cols):
    """Per query: (|E & O| int32, mass(E) fp64, mass(O) fp64) of two sorted CSR index sets
    under the fp64 score rows (dsv_set_stats_f64)."""
    _require_cuda(scores, e_ptr, o_ptr)
    _need_f64(scores)
    Q = scores.shape[0]
    inter = torch.empty((Q,), device=scores.device, dtype=torch.int32)
    em = torch.empty((Q,), device=scores.device, dtype=_F64)
    om = torch.empty((Q,), device=scores.device, dtype=_F64)
    _lib.call("dsv_set_stats_f64", _ptr(scores), scores.stride(0), Q, _ptr(e_ptr), _ptr(e_cols),
              _ptr(o_ptr), _ptr(o_cols), _ptr(inter), _ptr(em), _ptr(om), _stream())
    return inter, em, om
