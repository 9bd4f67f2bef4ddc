"""Autograd entry points (reference pkg/src/dynsparse/trainer.py:104-118).

* `group_sparse_attention(q, k, v, plan, idx, kcount)` — [H, L, D] bf16, one
  critical-KV list per (head, voxel group); forward K3f / backward K3b on
  tcgen05. This is the north_star operator (per-head index sets).
* `block_sparse_attention(q, k, v, idx)` — the exact `_Block.attention(x, idx)`
  formulation: q, k, v [B, H, S, d_k], idx [B, S, k] key ids shared across heads
  (trainer.py:111-117), gradients only through the gathered pairs. Any d_k and
  index pattern; fp32 CUDA-core kernels with fp32 atomics for dK/dV.
"""

from __future__ import annotations

import math

import torch

from . import ops


class _GroupSparseAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, grp_rows, grp_size, idx, kcount, kcount_hg, scale, tile_grp):
        out, lse = ops.sparse_fwd(q, k, v, grp_rows, grp_size, idx, kcount, scale, kcount_hg,
                                  tile_grp=tile_grp)
        ctx.save_for_backward(q, k, v, out, lse, grp_rows, grp_size, idx, kcount)
        ctx.kcount_hg = kcount_hg
        ctx.tile_grp = tile_grp
        ctx.scale = scale
        return out

    @staticmethod
    def backward(ctx, dout):
        q, k, v, out, lse, grp_rows, grp_size, idx, kcount = ctx.saved_tensors
        dq, dk32, dv32 = ops.sparse_bwd(q, k, v, out, dout.contiguous(), lse, grp_rows, grp_size,
                                        idx, kcount, ctx.scale, kcount_hg=ctx.kcount_hg,
                                        tile_grp=ctx.tile_grp)
        return (dq, ops.f32_to_bf16(dk32), ops.f32_to_bf16(dv32),
                None, None, None, None, None, None, None)


def group_sparse_attention(q, k, v, plan, idx, kcount, kcount_hg=None, scale=None):
    """Differentiable group-tiled sparse attention. q, k, v: [H, L, D] bf16 CUDA."""
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[-1])
    rows, size, tg = plan.tile_tables(q.device)
    return _GroupSparseAttention.apply(q.contiguous(), k.contiguous(), v.contiguous(), rows, size,
                                       idx, kcount, kcount_hg, float(scale), tg)


class _RowsSparseAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, ptr, cols, scale):
        out, lse = ops.rows_fwd(q, k, v, ptr, cols, scale)
        ctx.save_for_backward(q, k, v, out, lse, ptr, cols)
        ctx.scale = scale
        return out.to(q.dtype)

    @staticmethod
    def backward(ctx, dout):
        q, k, v, out, lse, ptr, cols = ctx.saved_tensors
        dq, dk, dv = ops.rows_bwd(q, k, v, out, lse, dout.to(q.dtype).contiguous(), ptr, cols,
                                  ctx.scale)
        return dq.to(q.dtype), dk.to(k.dtype), dv.to(v.dtype), None, None, None


def block_sparse_attention(q, k, v, idx):
    """`_Block.attention` sparse path: q, k, v [B, H, S, d_k], idx [B, S, k] -> [B, H, S, d_k]."""
    if q.dim() != 4:
        raise ValueError("q, k, v must be [B, H, S, d_k]")
    b, h, s, dk = q.shape
    if idx.shape[0] != b or idx.shape[1] != s:
        raise ValueError(f"idx must be [B={b}, S={s}, k], got {tuple(idx.shape)}")
    kk = idx.shape[2]
    if kk < 1:
        raise ValueError("every query needs at least one selected index")
    scale = 1.0 / math.sqrt(dk)
    dev = q.device
    outs = []
    for i in range(b):
        # the same [S, k] lists for every head -> one CSR over (head, query)
        cols = idx[i].to(device=dev, dtype=torch.int32).reshape(-1).repeat(h)
        ptr = torch.arange(0, h * s * kk + 1, kk, device=dev, dtype=torch.int64)
        outs.append(_RowsSparseAttention.apply(q[i].contiguous(), k[i].contiguous(),
                                               v[i].contiguous(), ptr, cols, scale))
    return torch.stack(outs)
