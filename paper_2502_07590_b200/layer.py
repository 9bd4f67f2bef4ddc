"""One DSV dynamic-sparsity attention layer on a single B200.

The hot path of BASELINE.json's north_star, end to end on device:

  K1a  project      P = X . Wt^T          [L, 2*H*r]  (Q_lr | K_lr for all heads)   tcgen05
  K1b  scores       S_h = Q_lr[proxies] . K_lr^T  [H, G, L] fp32                 tcgen05
  K2   select       exact top-k_h per (head, group) row -> idx [H, G, k_max]      CUDA cores
  K3f  sparse fwd   O, LSE over the selected KV of each group tile                 tcgen05/TMEM
  K3b  sparse bwd   dQ, dK, dV (dK/dV scatter-added in fp32)                       tcgen05/TMEM

Reference mapping (pkg/src/dynsparse): predictor.py:217-259 estimate_critical
(per head: project + top-k on the proxy rows, grouping.py:184-193), then
grouping.py:196-216 grouped_sparse_attention and its autograd
(trainer.py:110-117). Per-head k = k_from_sparsity(s_h, L)
(selection.py:60-67); heads may use different sparsities.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .grid import TokenGrid
from .grouping import VoxelGroupPlan, build_groups
from .selection import k_from_sparsity


@dataclass
class SelectedKV:
    """Device index lists: idx int32 [H, G, k_max] ascending, kcount int32 [H]."""

    idx: torch.Tensor
    kcount: torch.Tensor
    thresholds: torch.Tensor   # fp32 [H, G], k-th largest approximate score
    ks: list


class DSVAttentionLayer:
    """Predictor + selection + sparse attention for one layer, device resident."""

    def __init__(self, grid: TokenGrid, heads: int, head_dim: int, d_lr: int = 16,
                 voxel=(8, 4, 4), sparsity=0.9, device="cuda", groups=None):
        """groups: optional subset of the plan's voxel groups this layer serves (a
        sequence shard under hybrid CP); queries/keys stay addressed by global token."""
        self.grid = grid
        self.H = int(heads)
        self.D = int(head_dim)
        self.r = int(d_lr)
        self.device = torch.device(device)
        self.plan: VoxelGroupPlan = build_groups(grid, voxel)
        self.L = grid.size
        sp = np.broadcast_to(np.asarray(sparsity, dtype=np.float64), (self.H,))
        self.ks = [k_from_sparsity(float(s), self.L) for s in sp]
        self.kcount = torch.tensor(self.ks, dtype=torch.int32, device=self.device)
        self.k_max = max(self.ks)
        # query tiles of 128 (groups of the (8,8,4) / (8,8,8) ladder shapes span several tiles
        # sharing their index row, tile_grp: tile -> group); a `groups` subset keeps its tiles
        self.grp_rows, self.grp_size, self.tile_grp = self.plan.tile_tables(self.device, groups)
        self.proxies = self.plan.proxies_tensor(self.device)
        self._G = self.plan.n_groups
        if groups is not None:
            sel = torch.as_tensor(np.asarray(groups, dtype=np.int64), device=self.device)
            self.proxies = self.proxies[sel].contiguous()
            self._G = int(sel.numel())
        self.scale = 1.0 / math.sqrt(self.D)

    @property
    def G(self) -> int:
        return self._G

    # ------------------------------------------------------------- predictor
    def predictor_weights(self, seed: int = 0) -> torch.Tensor:
        """Random per-head W_q, W_k (PredictorParams.initialize: N(0, 1/sqrt(d)))
        stacked transposed as Wt [2*H*r, H*D] bf16."""
        g = torch.Generator(device="cpu").manual_seed(seed)
        d_model = self.H * self.D
        wt = torch.randn((2 * self.H * self.r, d_model), generator=g) / math.sqrt(d_model)
        return wt.to(torch.bfloat16).to(self.device)

    def select(self, x: torch.Tensor, wt: torch.Tensor, return_scores: bool = False):
        """K1a + K1b + K2: critical-KV index lists per (head, group)."""
        H, r, L = self.H, self.r, self.L
        p = ops.project(x, wt)                                   # [L, 2 H r] bf16
        qp = ops.gather_rows(p[:, : H * r], self.proxies)        # [G, H r] proxy rows
        qp = qp.view(self.G, H, r).permute(1, 0, 2)              # [H, G, r] (strided view)
        k_lr = p[:, H * r:].view(L, H, r).permute(1, 0, 2)       # [H, L, r] (strided view)
        return self._scores_topk(qp, k_lr, return_scores)

    def select_from_lowrank(self, q_lr: torch.Tensor, k_lr: torch.Tensor,
                            return_scores: bool = False):
        """K1b + K2 from per-head low-rank projections q_lr, k_lr [H, L, r] (bf16)."""
        H, r, L, G = self.H, self.r, self.L, self.G
        # proxy rows of every head: rows (h * L + proxy) of q_lr viewed as [H * L, r]
        key = ("prows", str(q_lr.device))
        if key not in self.__dict__:
            rows = (torch.arange(H, device=q_lr.device, dtype=torch.int32)[:, None] * L
                    + self.proxies[None, :]).reshape(-1)
            self.__dict__[key] = rows
        q2 = q_lr if q_lr.stride(0) == L * q_lr.stride(1) else q_lr.contiguous()
        qp = ops.gather_rows(q2.reshape(H * L, r) if q2.is_contiguous() else
                             torch.as_strided(q2, (H * L, r), (q2.stride(1), 1)),
                             self.__dict__[key]).view(H, G, r)
        return self._scores_topk(qp, k_lr, return_scores)

    def _scores_topk(self, qp, k_lr, return_scores):
        H, L, G = self.H, self.L, self.G
        hc = H if return_scores else self.score_heads_per_chunk()
        if not return_scores and self.fused_select():
            # K1b + K2 fused: scores recomputed on tcgen05 per pass, never stored; the layer
            # keeps its single-pass workspace alive (captured graphs hold its address)
            self.__dict__.setdefault("_sel_ws", ops.select_workspace(H, G, L, self.k_max, 0,
                                                                     qp.device))
            idx, thr = ops.select_fused(qp, k_lr, self.kcount, self.k_max)
            scores = None
        elif hc >= H:
            scores = ops.gemm_bf16(qp, k_lr, torch.float32)          # [H, G, L] fp32
            idx, thr = ops.topk_rows(scores.view(H * G, L), self.kcount, G, self.k_max)
        else:
            # long sequences (c5: 8.6 GB of scores per head): score and select hc heads at a
            # time through one reused buffer; the index lists land in place
            dev = qp.device
            idx = torch.empty((H * G, self.k_max), device=dev, dtype=torch.int32)
            thr = torch.empty((H * G,), device=dev, dtype=torch.float32)
            buf = torch.empty((hc, G, L), device=dev, dtype=torch.float32)
            for h0 in range(0, H, hc):
                h1 = min(H, h0 + hc)
                sc = ops.gemm_bf16(qp[h0:h1], k_lr[h0:h1], torch.float32, out=buf[: h1 - h0])
                ops.topk_rows(sc.view(-1, L), self.kcount[h0:h1], G, self.k_max,
                              out=(idx[h0 * G:h1 * G], thr[h0 * G:h1 * G]))
            scores = None
        sel = SelectedKV(idx.view(H, G, self.k_max), self.kcount, thr.view(H, G), self.ks)
        return (sel, scores) if return_scores else sel

    def fused_select(self) -> bool:
        """Fused K1b + K2 (select_fused.cu; r <= 16) where it measured faster than scores
        GEMM + top-k (tools/select_bench.py on one B200, single-pass mode, occupancy-sized
        key-range split): from 32 row tiles of 128 proxies (c2: 24 heads 0.47 vs 0.87 ms, 12
        heads 0.34 vs 0.48), or 16 at L >= 65536 (L = 131072, 2 heads: 0.73 vs 1.24 ms). With
        fewer tiles the fused kernel's sample passes and cluster merges are exposed (c2, 6
        heads: 0.28 vs 0.28 ms alone, and 2.12 vs 2.09 ms per 4-GPU step; 3 heads: 0.26 vs
        0.17 ms). DSV_FUSED_SELECT=1 / 0 forces either path."""
        if self.r > 16:
            return False
        env = os.environ.get("DSV_FUSED_SELECT", "auto")
        if env in ("0", "1"):
            return env == "1"
        tiles = self.H * ((self.G + 127) // 128)
        return tiles >= 32 or (tiles >= 16 and self.L >= 65536)

    def score_heads_per_chunk(self) -> int:
        """Heads scored per pass: the fp32 score matrices stay under DSV_SCORE_BYTES (16 GiB)."""
        per_head = self.G * self.L * 4
        budget = int(os.environ.get("DSV_SCORE_BYTES", str(16 << 30)))
        return max(1, min(self.H, budget // per_head))

    # ------------------------------------------------------------- attention
    def forward(self, q, k, v, sel: SelectedKV, prepare_backward: bool = True, out_rows=None):
        """Sparse forward. prepare_backward: the kernel also zeroes the layer's dK/dV
        accumulators for the coming backward (HBM writes hidden under the gather-bound
        forward instead of a separate fill pass). out_rows: (tab, n, chunk) row addresses the
        epilogue also stores O at (the token owners under head-parallel CP)."""
        zero = None
        if prepare_backward:
            zero = self._accumulators(k.shape[1], k.device)
            self._acc_zeroed = True
        return ops.sparse_fwd(q, k, v, self.grp_rows, self.grp_size, sel.idx, sel.kcount,
                              self.scale, zero=zero, tile_grp=self.tile_grp, out_rows=out_rows)

    def backward(self, q, k, v, out, lse, dout, sel: SelectedKV, dk_acc=None, dv_acc=None,
                 kernel_done=None, dq_rows=None, dkdv_rows=None):
        """-> (dq, dk, dv) bf16. Without caller accumulators the layer's own are used (zeroed
        by the preceding forward, or here if that did not happen). dq_rows / dkdv_rows:
        (tab, n, chunk) row addresses dQ / (dK, dV) go to instead (the token owners under
        head-parallel CP); the corresponding results are then None."""
        if dk_acc is None:
            acc = self._accumulators(k.shape[1], k.device)
            if not getattr(self, "_acc_zeroed", False):
                acc.zero_()
            self._acc_zeroed = False
            dk_acc, dv_acc = acc[0], acc[1]
        else:
            dk_acc.zero_()
            dv_acc.zero_()
        if os.environ.get("DSV_BWD_CONVERT", "1") != "0":
            # the backward kernel converts dK / dV to bf16 itself, in its tail (CTAs that run
            # out of tiles convert the heads already finished); DSV_BWD_CONVERT=0: separately
            dkdv = None
            if dkdv_rows is None:
                dkdv = torch.empty((2, self.H, k.shape[1], self.D), device=k.device,
                                   dtype=torch.bfloat16)
            dq, _, _ = ops.sparse_bwd(q, k, v, out, dout, lse, self.grp_rows, self.grp_size,
                                      sel.idx, sel.kcount, self.scale, dk_acc, dv_acc,
                                      tile_grp=self.tile_grp, dq_rows=dq_rows, dkdv_out=dkdv,
                                      dkdv_rows=dkdv_rows)
            if kernel_done is not None:
                kernel_done.record()
            dq = None if dq_rows is not None else dq
            return (dq, None, None) if dkdv is None else (dq, dkdv[0], dkdv[1])
        dq, dk32, dv32 = ops.sparse_bwd(q, k, v, out, dout, lse, self.grp_rows, self.grp_size,
                                        sel.idx, sel.kcount, self.scale, dk_acc, dv_acc,
                                        tile_grp=self.tile_grp, dq_rows=dq_rows)
        if kernel_done is not None:          # optional CUDA event after the kernel (timing)
            kernel_done.record()
        if dkdv_rows is not None:
            ops.f32_to_bf16_rows(dk32, dkdv_rows[0])
            ops.f32_to_bf16_rows(dv32, dkdv_rows[1])
            return (None if dq_rows is not None else dq), None, None
        return (None if dq_rows is not None else dq), ops.f32_to_bf16(dk32), ops.f32_to_bf16(dv32)

    def _accumulators(self, n_keys: int, device):
        """The layer's fp32 dK/dV accumulators [2, H, n_keys, D] (one contiguous buffer)."""
        key = (int(n_keys), str(device))
        if self.__dict__.get("_acc_key") != key:
            self._acc = torch.empty((2, self.H, int(n_keys), self.D), device=device,
                                    dtype=torch.float32)
            self._acc_key = key
            self._acc_zeroed = False
        return self._acc

    def step(self, x, wt, q, k, v, dout, dk_acc=None, dv_acc=None):
        """One fwd+bwd pass of the layer (the bench's unit of work)."""
        sel = self.select(x, wt)
        out, lse = self.forward(q, k, v, sel, prepare_backward=dk_acc is None)
        dq, dk, dv = self.backward(q, k, v, out, lse, dout, sel, dk_acc, dv_acc)
        return out, dq, dk, dv

    # ------------------------------------------------------------- accounting
    def pairs(self) -> int:
        """(query, key) pairs scored per pass: sum over this layer's query groups and heads."""
        nq = int(self.grp_size.sum().item()) if self._G != self.plan.n_groups else self.L
        return sum(nq * kh for kh in self.ks)

    def work(self) -> dict:
        """Algorithmic work per layer pass."""
        H, r, L, G, D = self.H, self.r, self.L, self.G, self.D
        pairs = self.pairs()
        return {
            "projection_flops": 2 * L * (H * D) * (2 * r * H),
            "estimation_flops": 2 * H * G * L * r,
            "topk_bytes": H * G * (L * 4 + 4) + sum(G * kh * 4 for kh in self.ks),
            "fwd_flops": 4 * pairs * D,
            "bwd_flops": 10 * pairs * D,
        }


class HostPipeline:
    """Runs a device step over host-resident batches: H2D of batch i+1 and D2H of step i's
    results overlap step i+1 / step i on two copy streams.

    Two device input buffer sets filled from pinned host memory on the H2D stream; each
    step's result tensors are copied back into one of two pinned host output sets on the D2H
    stream (full-duplex PCIe: both directions at once). Yields each step's host output set;
    its contents are valid once `drain()` (or a later synchronize) returns.
    """

    def __init__(self, like, device):
        dev = torch.device(device)
        self.bufs = [[torch.empty(t.shape, dtype=t.dtype, device=dev) for t in like] for _ in range(2)]
        self.copy = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.ready = [torch.cuda.Event(), torch.cuda.Event()]
        self.free = [None, None]
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in like)
        self.d2h_bytes = 0
        self.host_out = [None, None]
        self.held = [None, None]            # device results still being copied out
        self.fetched = [None, None]         # D2H completion of each slot

    def _stage(self, slot, host):
        with torch.cuda.stream(self.copy):
            if self.free[slot] is not None:
                self.copy.wait_event(self.free[slot])
            for src, dst in zip(host, self.bufs[slot]):
                if not src.is_pinned():
                    raise ValueError("HostPipeline expects pinned host tensors")
                dst.copy_(src, non_blocking=True)
            self.ready[slot].record(self.copy)

    def _fetch(self, slot, res, reused: bool = False):
        """D2H of the step's result tensors into pinned host set `slot` on the D2H stream. The
        device tensors stay referenced until the compute stream has waited for the copy (the
        slot's next step), so the allocator never hands their memory out while it is read.
        reused: the results are views of buffers the next step overwrites (head-parallel CP
        returns views of its peer buffers) — they are first copied on the device."""
        res = [t for t in (res if isinstance(res, (tuple, list)) else (res,)) if torch.is_tensor(t)]
        if reused:
            res = [t.clone() for t in res]
        if self.host_out[slot] is None:
            self.host_out[slot] = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in res]
            self.d2h_bytes = sum(t.numel() * t.element_size() for t in res)
        self.d2h.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.d2h):
            for t, h in zip(res, self.host_out[slot]):
                h.copy_(t, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.d2h)
        self.held[slot] = res
        self.fetched[slot] = ev
        return self.host_out[slot]

    def drain(self):
        """Make the current stream wait for every issued D2H copy."""
        torch.cuda.current_stream().wait_stream(self.d2h)

    def run(self, step, batches, fetch: bool = True, reused: bool = False):
        it = iter(batches)
        nxt = next(it, None)
        slot = 0
        if nxt is not None:
            self._stage(slot, nxt)
        while nxt is not None:
            nxt = next(it, None)
            if nxt is not None:
                self._stage(slot ^ 1, nxt)
            cur = torch.cuda.current_stream()
            cur.wait_event(self.ready[slot])
            if self.fetched[slot] is not None:      # the slot's previous results are copied out
                cur.wait_event(self.fetched[slot])
                self.held[slot] = None
            res = step(*self.bufs[slot])
            ev = torch.cuda.Event()
            ev.record(cur)
            self.free[slot] = ev
            yield self._fetch(slot, res, reused) if fetch else res
            slot ^= 1
