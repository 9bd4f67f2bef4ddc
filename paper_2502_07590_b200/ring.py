"""Ring KV pass for dense residual heads under sequence-wise context parallelism.

SURVEY §2.1 ("ring attention / blockwise KV ring": absent from the reference, required by
the north_star: "ring KV exchange only for residual dense blocks") and §8(e). A head that
the dispatcher runs dense (`dispatcher.decide` -> "full", src/dispatcher.py:235-260) gains
nothing from selective KV gathering: every query needs every key, so the SCP group of g_s
ranks that share the head passes the K/V chunks around a ring instead, one hop per rank,
with the transfer of the next chunk overlapping the attention on the current one. The
semantics are the reference's dense attention (`full_attention`, src/attention.py:95-109,
pinned by tests/test_cpsim.py:75-88): softmax over all keys of q.k / sqrt(d).

Forward: hop t attends the local queries to the visiting chunk with the tcgen05 kernel
(every key of the chunk selected) and merges the partial rows by their log-sum-exp
(`dsv_ring_lse_merge`). Backward: with the final O and LSE every (query, key) term is
local, so each hop adds dQ (fp32, `dsv_ring_accum_bf16`) and the visiting chunk's dK/dV;
the latter travel with the ring as fp32 accumulators (`dsv_ring_accum_f32` folds one hop's
atomically-accumulated part into the accumulator and re-zeroes the part) and arrive home
after the last hop. Per rank and direction the ring moves (g_s - 1) K/V chunks forward
and g_s fp32 dK/dV accumulators backward (ledger phases "ring_kv", "ring_kv_bwd",
"ring_grad").

Transport: `torch.distributed.batch_isend_irecv` to the ring neighbours (NCCL P2P over
NVLink on the GPU box; gloo in the CPU tests). The per-hop device work is a `RingKernels`
object; the CPU tests substitute a float64 torch implementation of the same contract.
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist

from .grid import TokenGrid
from .grouping import build_groups

TILE = 128


class RingKernels:
    """The per-hop device work (libdsv kernels): queries tiled in 128-row groups, every key
    of the visiting chunk selected (the shared index row has stride 0 across groups)."""

    def __init__(self, n_queries: int, n_keys: int, heads: int, head_dim: int, scale=None,
                 device="cuda"):
        dev = torch.device(device)
        plan = build_groups(TokenGrid(1, 1, n_queries), (1, 1, min(TILE, n_queries)))
        self.grp_rows, self.grp_size = plan.tables(dev)
        self.G = plan.n_groups
        self.idx = torch.arange(n_keys, device=dev, dtype=torch.int32).expand(heads, self.G, n_keys)
        self.kcount = torch.full((heads,), n_keys, device=dev, dtype=torch.int32)
        self.scale = 1.0 / math.sqrt(head_dim) if scale is None else float(scale)

    def attend(self, q, k, v):
        from . import ops
        return ops.sparse_fwd(q, k, v, self.grp_rows, self.grp_size, self.idx, self.kcount, self.scale)

    def grad(self, q, k, v, out, dout, lse, dk_part, dv_part):
        from . import ops
        dq, _, _ = ops.sparse_bwd(q, k, v, out, dout, lse, self.grp_rows, self.grp_size, self.idx,
                                  self.kcount, self.scale, dk_part, dv_part)
        return dq

    @staticmethod
    def merge(acc, lse_in, lse_out, part, lse_part, first, out=None):
        from . import ops
        ops.ring_lse_merge(acc, lse_in, lse_out, part, lse_part, first, out)

    @staticmethod
    def accum_dq(acc, x, first, out=None):
        from . import ops
        ops.ring_accum_bf16(acc, x, first, out)

    @staticmethod
    def accum_kv(acc, part, first):
        from . import ops
        ops.ring_accum_f32(acc, part, first)

    @staticmethod
    def to_bf16(x):
        from . import ops
        return ops.f32_to_bf16(x)


class RingKV:
    """Dense attention of this rank's query chunk against the K/V chunks of every rank of
    `group`, passed around a ring. Inputs per rank: q, k, v [H, Lc, D] (this rank's chunk
    of the sequence, chunks in group-rank order). `kernels` defaults to `RingKernels`."""

    def __init__(self, group=None, kernels=None, ledger=None):
        self.group = group
        self.n = dist.get_world_size(group) if dist.is_initialized() else 1
        self.pos = dist.get_rank(group) if dist.is_initialized() else 0
        glob = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))
        self.next = glob((self.pos + 1) % self.n)
        self.prev = glob((self.pos - 1) % self.n)
        self.kernels = kernels
        self.ledger = ledger
        self._cache = {}

    def _k(self, q, k):
        if self.kernels is not None:
            return self.kernels
        key = (q.shape, k.shape[1], q.device)
        if key not in self._cache:
            self._cache[key] = RingKernels(q.shape[1], k.shape[1], q.shape[0], q.shape[2],
                                           device=q.device)
        return self._cache[key]

    def _shift(self, pairs, phase):
        """pairs: [(send tensor, recv tensor)]: send to next, receive from prev (in order)."""
        ops = []
        for s, r in pairs:
            ops.append(dist.P2POp(dist.isend, s, self.next, self.group))
            ops.append(dist.P2POp(dist.irecv, r, self.prev, self.group))
            if self.ledger is not None:
                nb = s.numel() * s.element_size()
                self.ledger.add(phase, nb, nb)
        return dist.batch_isend_irecv(ops) if ops else []

    def _kv_buffers(self, k, v):
        """Two receive buffers used alternately (the caller's k, v are only ever sent)."""
        m = min(self.n - 1, 2)
        return [(torch.empty_like(k), torch.empty_like(v)) for _ in range(m)]

    @staticmethod
    def _wait(reqs):
        for r in reqs:
            r.wait()

    def forward(self, q, k, v):
        """-> (out bf16 [H, Lc, D], lse fp32 [H, Lc], log2 domain of the scaled logits)."""
        K = self._k(q, k)
        n = self.n
        H, Lc, D = q.shape
        cur = (k, v)
        bufs = self._kv_buffers(k, v)
        acc = torch.empty((H, Lc, D), dtype=torch.float32, device=q.device)
        lse = [torch.empty((H, Lc), dtype=torch.float32, device=q.device) for _ in range(min(n, 2))]
        out = torch.empty_like(q)
        for t in range(n):
            reqs = self._shift(list(zip(cur, bufs[t % 2])), "ring_kv") if t < n - 1 else []
            o_t, l_t = K.attend(q, *cur)
            K.merge(acc, lse[(t - 1) % 2] if t else None, lse[t % 2], o_t, l_t, t == 0,
                    out if t == n - 1 else None)
            self._wait(reqs)
            if t < n - 1:
                cur = bufs[t % 2]
        return out, lse[(n - 1) % 2]

    def backward(self, q, k, v, out, lse, dout):
        """-> (dq, dk, dv) bf16 [H, Lc, D] for this rank's chunk."""
        K = self._k(q, k)
        n = self.n
        H, Lc, D = q.shape
        dev = q.device
        cur = (k, v)
        bufs = self._kv_buffers(k, v)
        part = torch.zeros((2, H, Lc, D), dtype=torch.float32, device=dev)
        accs = [torch.empty((2, H, Lc, D), dtype=torch.float32, device=dev) for _ in range(min(n, 2))]
        dq_acc = torch.empty((H, Lc, D), dtype=torch.float32, device=dev)
        dq = torch.empty_like(q)
        for t in range(n):
            pairs = list(zip(cur, bufs[t % 2])) if t < n - 1 else []
            reqs = self._shift(pairs, "ring_kv_bwd")
            if t >= 1:   # the accumulator of chunk (pos - t) arrives while this hop computes
                reqs += self._shift([(accs[(t - 1) % 2], accs[t % 2])], "ring_grad")
            dq_t = K.grad(q, *cur, out, dout, lse, part[0], part[1])
            K.accum_dq(dq_acc, dq_t, t == 0, dq if t == n - 1 else None)
            self._wait(reqs)
            K.accum_kv(accs[t % 2], part, t == 0)
            if t < n - 1:
                cur = bufs[t % 2]
        final = accs[0]
        if n > 1:    # the last accumulator goes home
            self._wait(self._shift([(accs[(n - 1) % 2], accs[n % 2])], "ring_grad"))
            final = accs[n % 2]
        return dq, K.to_bf16(final[0]), K.to_bf16(final[1])

    def expected_bytes(self, heads: int, chunk: int, head_dim: int, elem: int = 2,
                       acc_elem: int = 4) -> dict:
        """Bytes one rank sends per phase (it receives the same)."""
        kv = 2 * heads * chunk * head_dim
        return {"ring_kv": (self.n - 1) * kv * elem, "ring_kv_bwd": (self.n - 1) * kv * elem,
                "ring_grad": (self.n if self.n > 1 else 0) * kv * acc_elem}
