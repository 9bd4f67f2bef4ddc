"""Sparsity-aware head-parallel context parallelism over NCCL (HCP).

Executes the reference's Algorithm 1 HCP phases (pkg/src/dynsparse/cpsim.py:
125-161 `load_balance_hcp`, 284-299 output redistribution; byte model
cpmodel.py:213-223 `hcp_comm`) with real ranks, one process per GPU:

  1. each rank holds a contiguous chunk of L/N tokens for every head;
  2. the predictor projection runs on the local chunk (K1a);
  3. uneven all-to-all (NCCL, torch.distributed.all_to_all_single): every rank
     receives the full sequence of the heads `balance_heads` assigned to it
     (Q, K, V, Q_lr, K_lr; plus dO for the backward), head re-balancing by
     per-head sparsity so the skewed (1 - s_h) loads even out;
  4. local K1b/K2/K3 on the owned heads;
  5. the reverse all-to-all returns O (and dQ, dK, dV) to the token owners.

Packing for the exchange is a row gather (dsv_gather_rows) on CUDA tensors.
Every message size is recorded in a ledger with the reference's phase names so
the bytes can be checked against `hcp_comm` exactly (tests/test_cp_gloo.py
runs the protocol with world_size 2 on the gloo backend).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import cpmodel

PHASES = ("hcp_fwd", "scp_index_exchange", "scp_kv", "output_redistribute", "hcp_bwd_in",
          "hcp_bwd_out")


@dataclass
class Ledger:
    """Bytes this rank sends/receives per phase (cpsim.py:43-71, per rank)."""

    sent: dict = field(default_factory=dict)
    received: dict = field(default_factory=dict)

    def add(self, phase: str, sent: int, received: int) -> None:
        if phase not in PHASES:
            raise ValueError(f"unknown phase {phase!r}")
        self.sent[phase] = self.sent.get(phase, 0) + int(sent)
        self.received[phase] = self.received.get(phase, 0) + int(received)


def _gather_rows(src2d: torch.Tensor, rows: torch.Tensor) -> torch.Tensor:
    if src2d.is_cuda:
        from . import ops

        return ops.gather_rows(src2d, rows)
    return src2d.index_select(0, rows.long())


class HeadParallelExchange:
    """Head <-> sequence resharding for one process group (HCP, g_h = N)."""

    def __init__(self, n_heads: int, seq_len: int, assignment, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if seq_len % self.world:
            raise ValueError("sequence length must divide the rank count")
        self.H = int(n_heads)
        self.L = int(seq_len)
        self.chunk = self.L // self.world
        self.assignment = np.asarray(assignment, dtype=np.int64)
        if self.assignment.shape != (self.H,) or self.assignment.min() < 0 or self.assignment.max() >= self.world:
            raise ValueError("assignment must map every head to a rank")
        self.heads_of = [np.nonzero(self.assignment == r)[0] for r in range(self.world)]
        self.my_heads = self.heads_of[self.rank]
        self.ledger = Ledger()
        self._perm_cache = {}

    # ---------------------------------------------------------------- index maps
    def _send_rows(self, device) -> torch.Tensor:
        """Rows of a head-major [H * chunk] local tensor, grouped by destination."""
        key = ("send", str(device))
        if key not in self._perm_cache:
            rows = [h * self.chunk + t for r in range(self.world) for h in self.heads_of[r]
                    for t in range(self.chunk)]
            self._perm_cache[key] = torch.tensor(rows, dtype=torch.int32, device=device)
        return self._perm_cache[key]

    def _recv_rows(self, device) -> torch.Tensor:
        """Maps the received [src][my_heads][chunk] rows to [my_heads][L]."""
        key = ("recv", str(device))
        if key not in self._perm_cache:
            nh = len(self.my_heads)
            out = np.empty(nh * self.L, dtype=np.int64)
            for hi in range(nh):
                for r in range(self.world):
                    base = r * nh * self.chunk + hi * self.chunk
                    out[hi * self.L + r * self.chunk: hi * self.L + (r + 1) * self.chunk] = \
                        base + np.arange(self.chunk)
            self._perm_cache[key] = torch.from_numpy(out.astype(np.int32)).to(device)
        return self._perm_cache[key]

    def _inverse_rows(self, device):
        """[my_heads][L] rows grouped by destination rank (reverse exchange)."""
        key = ("inv", str(device))
        if key not in self._perm_cache:
            nh = len(self.my_heads)
            rows = [hi * self.L + r * self.chunk + t for r in range(self.world) for hi in range(nh)
                    for t in range(self.chunk)]
            self._perm_cache[key] = torch.tensor(rows, dtype=torch.int32, device=device)
        return self._perm_cache[key]

    def _back_rows(self, device):
        """Received [src][src_heads][chunk] rows -> head-major [H][chunk]."""
        key = ("back", str(device))
        if key not in self._perm_cache:
            pos = np.empty(self.H * self.chunk, dtype=np.int64)
            off = 0
            for r in range(self.world):
                for h in self.heads_of[r]:
                    pos[h * self.chunk: (h + 1) * self.chunk] = off + np.arange(self.chunk)
                    off += self.chunk
            self._perm_cache[key] = torch.from_numpy(pos.astype(np.int32)).to(device)
        return self._perm_cache[key]

    # ---------------------------------------------------------------- exchanges
    def to_heads(self, local: torch.Tensor, phase: str = "hcp_fwd") -> torch.Tensor:
        """[H, chunk, W] (all heads, my tokens) -> [my_heads, L, W] (my heads, all tokens)."""
        H, chunk, W = local.shape
        if H != self.H or chunk != self.chunk:
            raise ValueError(f"expected [{self.H}, {self.chunk}, *], got {tuple(local.shape)}")
        flat = local.reshape(H * chunk, W)
        send = _gather_rows(flat, self._send_rows(local.device))
        nh = len(self.my_heads)
        recv = torch.empty((self.world * nh * chunk, W), dtype=local.dtype, device=local.device)
        in_split = [len(self.heads_of[r]) * chunk for r in range(self.world)]
        out_split = [nh * chunk] * self.world
        dist.all_to_all_single(recv, send, out_split, in_split, group=self.group)
        es = local.element_size() * W
        self.ledger.add(phase, (sum(in_split) - in_split[self.rank]) * es,
                        (sum(out_split) - out_split[self.rank]) * es)
        return _gather_rows(recv, self._recv_rows(local.device)).view(nh, self.L, W)

    def to_tokens(self, mine: torch.Tensor, phase: str = "output_redistribute") -> torch.Tensor:
        """[my_heads, L, W] -> [H, chunk, W] (inverse of to_heads)."""
        nh, L, W = mine.shape
        if nh != len(self.my_heads) or L != self.L:
            raise ValueError("shape does not match this rank's head plan")
        flat = mine.reshape(nh * L, W)
        send = _gather_rows(flat, self._inverse_rows(mine.device))
        recv = torch.empty((self.H * self.chunk, W), dtype=mine.dtype, device=mine.device)
        in_split = [nh * self.chunk] * self.world
        out_split = [len(self.heads_of[r]) * self.chunk for r in range(self.world)]
        dist.all_to_all_single(recv, send, out_split, in_split, group=self.group)
        es = mine.element_size() * W
        self.ledger.add(phase, (sum(in_split) - in_split[self.rank]) * es,
                        (sum(out_split) - out_split[self.rank]) * es)
        return _gather_rows(recv, self._back_rows(mine.device)).view(self.H, self.chunk, W)

    def expected_hcp_bytes(self, d: int, elem_width: int) -> float:
        """hcp_comm for this rank (Q, K, V in + O back), cpmodel.py:213-223."""
        return cpmodel.hcp_comm(self.H, len(self.my_heads), self.L, d, self.world, elem_width)


def plan_heads(sparsities, seq_len: int, head_dim: int, world: int, balanced: bool = True):
    """Head -> rank assignment: sparsity-aware `balance_heads` or the contiguous split."""
    if not balanced:
        return cpmodel.contiguous_heads(len(sparsities), world).assignment
    loads = cpmodel.head_loads(sparsities, seq_len, head_dim)
    return cpmodel.balance_heads(loads, world).assignment


class HeadParallelDSV:
    """The DSV layer under HCP: sequence-sharded in, sequence-sharded out."""

    def __init__(self, grid, heads: int, head_dim: int, d_lr: int = 16, voxel=(8, 4, 4),
                 sparsity=0.9, balanced: bool = True, group=None, device="cuda"):
        from .layer import DSVAttentionLayer

        self.world = dist.get_world_size(group)
        sp = np.broadcast_to(np.asarray(sparsity, dtype=np.float64), (heads,)).copy()
        self.assignment = plan_heads(sp, grid.size, head_dim, self.world, balanced)
        self.ex = HeadParallelExchange(heads, grid.size, self.assignment, group)
        self.H, self.D, self.r = heads, head_dim, d_lr
        mine = self.ex.my_heads
        self.local = DSVAttentionLayer(grid, len(mine), head_dim, d_lr, voxel, sp[mine], device)

    def step(self, x_local, wt, q, k, v, dout):
        """x_local [L/N, H*D]; q, k, v, dout [H, L/N, D] -> (out, dq, dk, dv) [H, L/N, D]."""
        from . import ops

        H, r = self.H, self.r
        p = ops.project(x_local, wt)                                   # [L/N, 2 H r]
        plr = p.view(-1, 2, H, r).permute(2, 0, 1, 3).reshape(H, -1, 2 * r)   # [H, L/N, 2r]
        # one exchange for Q | K | V | Q_lr K_lr (same head plan)
        packed = torch.cat([q, k, v, plr.contiguous()], dim=2)         # [H, L/N, 3D + 2r]
        mine = self.ex.to_heads(packed, "hcp_fwd")                     # [h, L, 3D + 2r]
        D = self.D
        ql, kl, vl = (mine[:, :, i * D:(i + 1) * D].contiguous() for i in range(3))
        lr = mine[:, :, 3 * D:]
        sel = self.local.select_from_lowrank(lr[:, :, :r], lr[:, :, r:])
        out, lse = self.local.forward(ql, kl, vl, sel)
        dout_m = self.ex.to_heads(dout, "hcp_bwd_in")
        dq, dk, dv = self.local.backward(ql, kl, vl, out, lse, dout_m, sel)
        back = self.ex.to_tokens(torch.cat([out, dq, dk, dv], dim=2), "hcp_bwd_out")
        return tuple(back[:, :, i * D:(i + 1) * D] for i in range(4))
