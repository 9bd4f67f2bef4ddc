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

import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, cpmodel

PHASES = ("hcp_fwd", "scp_index_exchange", "scp_kv", "output_redistribute", "hcp_bwd_in",
          "hcp_bwd_out", "scp_grad",   # scp_grad: dK/dV of gathered rows back to their owners
                                       # (the reference simulator is forward-only)
          "ring_kv", "ring_kv_bwd", "ring_grad")   # ring KV pass of dense heads (ring.py)


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


def _gather_into(src2d: torch.Tensor, rows: torch.Tensor, out2d: torch.Tensor) -> None:
    """out2d[j] = src2d[rows[j]] (row gather; dsv_gather_rows on CUDA tensors)."""
    if src2d.is_cuda:
        from . import ops

        ops.gather_rows(src2d, rows, out=out2d)
    else:
        out2d.copy_(src2d.index_select(0, rows.long()))


def _gather_rows(src2d: torch.Tensor, rows: torch.Tensor) -> torch.Tensor:
    out = torch.empty((rows.numel(), src2d.shape[1]), dtype=src2d.dtype, device=src2d.device)
    _gather_into(src2d, rows, out)
    return out


class HeadParallelExchange:
    """Head <-> sequence resharding for one process group (HCP, g_h = N).

    Several tensors travel in one packed all-to-all: each contributes a column
    range of the packed rows, gathered straight from its own layout.
    """

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
        self._maps = {}

    # ---------------------------------------------------------------- index maps
    def _send_ht(self):
        """(head, local token) of every packed send row, grouped by destination."""
        if "send_ht" not in self._maps:
            hh = np.concatenate([np.repeat(self.heads_of[r], self.chunk) for r in range(self.world)])
            tt = np.tile(np.arange(self.chunk), self.H)
            self._maps["send_ht"] = (hh, tt)
        return self._maps["send_ht"]

    def _rows(self, key, fn, device):
        k = (key, str(device))
        if k not in self._maps:
            self._maps[k] = torch.from_numpy(np.ascontiguousarray(fn()).astype(np.int32)).to(device)
        return self._maps[k]

    def send_rows_headmajor(self, device):
        hh, tt = self._send_ht()
        return self._rows("hm", lambda: hh * self.chunk + tt, device)

    def send_rows_lowrank(self, side: int, device):
        """Rows of P [chunk, 2, H, r] viewed as [chunk * 2H, r]: (t, side, h)."""
        hh, tt = self._send_ht()
        return self._rows(("lr", side), lambda: tt * 2 * self.H + side * self.H + hh, device)

    def _recv_rows(self, device):
        """Received [src][my_heads][chunk] rows -> [my_heads][L]."""
        def fn():
            nh = len(self.my_heads)
            out = np.empty(nh * self.L, dtype=np.int64)
            for hi in range(nh):
                for r in range(self.world):
                    base = r * nh * self.chunk + hi * self.chunk
                    out[hi * self.L + r * self.chunk: hi * self.L + (r + 1) * self.chunk] = \
                        base + np.arange(self.chunk)
            return out
        return self._rows("recv", fn, device)

    def _inverse_rows(self, device):
        """[my_heads][L] rows grouped by destination rank (reverse exchange)."""
        nh = len(self.my_heads)
        return self._rows("inv", lambda: np.array(
            [hi * self.L + r * self.chunk + t for r in range(self.world) for hi in range(nh)
             for t in range(self.chunk)], dtype=np.int64), device)

    def _back_rows(self, device):
        """Received [src][src_heads][chunk] rows -> head-major [H][chunk]."""
        def fn():
            pos = np.empty(self.H * self.chunk, dtype=np.int64)
            off = 0
            for r in range(self.world):
                for h in self.heads_of[r]:
                    pos[h * self.chunk: (h + 1) * self.chunk] = off + np.arange(self.chunk)
                    off += self.chunk
            return pos
        return self._rows("back", fn, device)

    # ---------------------------------------------------------------- exchanges
    def to_heads_packed(self, sources, phase: str = "hcp_fwd", async_op: bool = False):
        """sources: list of (src2d, send_rows) whose send rows enumerate (dst, head, t).

        Returns a handle; `finish(handle)` -> list of [my_heads, L, W_i] tensors.
        """
        dev = sources[0][0].device
        dtype = sources[0][0].dtype
        widths = [s.shape[1] for s, _ in sources]
        W = sum(widths)
        send = torch.empty((self.H * self.chunk, W), dtype=dtype, device=dev)
        off = 0
        for (src, rows), w in zip(sources, widths):
            _gather_into(src, rows, send[:, off:off + w])
            off += w
        nh = len(self.my_heads)
        recv = torch.empty((self.world * nh * self.chunk, W), dtype=dtype, device=dev)
        in_split = [len(self.heads_of[r]) * self.chunk for r in range(self.world)]
        out_split = [nh * self.chunk] * self.world
        work = dist.all_to_all_single(recv, send, out_split, in_split, group=self.group,
                                      async_op=async_op)
        es = send.element_size() * W
        self.ledger.add(phase, (sum(in_split) - in_split[self.rank]) * es,
                        (sum(out_split) - out_split[self.rank]) * es)
        return ("heads", work, recv, widths, send)

    def to_tokens_packed(self, tensors, phase: str = "output_redistribute", async_op: bool = False):
        """tensors: list of [my_heads, L, W_i] -> handle for list of [H, chunk, W_i]."""
        nh = len(self.my_heads)
        dev, dtype = tensors[0].device, tensors[0].dtype
        widths = [t.shape[2] for t in tensors]
        W = sum(widths)
        send = torch.empty((nh * self.L, W), dtype=dtype, device=dev)
        rows = self._inverse_rows(dev)
        off = 0
        for t, w in zip(tensors, widths):
            if t.shape[0] != nh or t.shape[1] != self.L:
                raise ValueError("shape does not match this rank's head plan")
            _gather_into(t.reshape(nh * self.L, w), rows, send[:, off:off + w])
            off += w
        recv = torch.empty((self.H * self.chunk, W), dtype=dtype, device=dev)
        in_split = [nh * self.chunk] * self.world
        out_split = [len(self.heads_of[r]) * self.chunk for r in range(self.world)]
        work = dist.all_to_all_single(recv, send, out_split, in_split, group=self.group,
                                      async_op=async_op)
        es = send.element_size() * W
        self.ledger.add(phase, (sum(in_split) - in_split[self.rank]) * es,
                        (sum(out_split) - out_split[self.rank]) * es)
        return ("tokens", work, recv, widths, send)

    def finish(self, handle):
        kind, work, recv, widths, _send = handle
        if work is not None:
            work.wait()
        dev = recv.device
        rows = self._recv_rows(dev) if kind == "heads" else self._back_rows(dev)
        lead = (len(self.my_heads), self.L) if kind == "heads" else (self.H, self.chunk)
        outs, off = [], 0
        for w in widths:
            outs.append(_gather_rows(recv[:, off:off + w], rows).view(*lead, w))
            off += w
        return outs

    # single-tensor conveniences (reference phase semantics)
    def to_heads(self, local: torch.Tensor, phase: str = "hcp_fwd") -> torch.Tensor:
        """[H, chunk, W] (all heads, my tokens) -> [my_heads, L, W] (my heads, all tokens)."""
        H, chunk, W = local.shape
        if H != self.H or chunk != self.chunk:
            raise ValueError(f"expected [{self.H}, {self.chunk}, *], got {tuple(local.shape)}")
        src = local.reshape(H * chunk, W)
        return self.finish(self.to_heads_packed([(src, self.send_rows_headmajor(local.device))], phase))[0]

    def to_tokens(self, mine: torch.Tensor, phase: str = "output_redistribute") -> torch.Tensor:
        """[my_heads, L, W] -> [H, chunk, W] (inverse of to_heads)."""
        return self.finish(self.to_tokens_packed([mine], phase))[0]

    def expected_hcp_bytes(self, d: int, elem_width: int) -> float:
        """hcp_comm for this rank (Q, K, V in + O back), cpmodel.py:213-223."""
        return cpmodel.hcp_comm(self.H, len(self.my_heads), self.L, d, self.world, elem_width)


class _CudaArray:
    """Minimal __cuda_array_interface__ view of raw device memory (int16 elements). `owner`
    is kept alive as long as any tensor made from this view (torch holds the interface object
    until the tensor's storage is released)."""

    def __init__(self, ptr: int, n: int, owner=None):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False),
                                         "version": 3, "strides": None}


class _PeerAlloc:
    """This rank's dsv_peer_alloc buffer; freed (after the device is idle) when the last
    tensor view of it is gone — step() results are views of it and may outlive the layer."""

    def __init__(self, ptr: int, device):
        self.ptr, self.device = ptr, device

    def __del__(self):
        try:
            torch.cuda.synchronize(self.device)
            _lib.load().dsv_peer_free(self.ptr)
        except Exception:
            pass


class _PeerBuffer:
    """This rank's peer-mapped device buffer plus every peer's, mapped into this process with
    CUDA IPC through libdsv (dsv_peer_alloc / dsv_peer_open; handles exchanged with
    all_gather_object). `tensor` is a bf16 view of the local buffer; `ptrs[r]` the address of
    rank r's buffer in this process."""

    def __init__(self, nbytes: int, group, device):
        import ctypes

        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        ptr, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
        with torch.cuda.device(device):
            _lib.call("dsv_peer_alloc", int(nbytes), ctypes.byref(ptr), handle)
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=group)
        self.ptrs, self._opened = [], []
        with torch.cuda.device(device):
            for r, h in enumerate(handles):
                if r == self.rank:
                    self.ptrs.append(int(ptr.value))
                    continue
                p = ctypes.c_void_p()
                _lib.call("dsv_peer_open", ctypes.create_string_buffer(h, 64), ctypes.byref(p))
                self.ptrs.append(int(p.value))
                self._opened.append(int(p.value))
        self._own = int(ptr.value)
        self._device = torch.device(device)
        alloc = _PeerAlloc(self._own, self._device)
        self.tensor = torch.as_tensor(_CudaArray(self._own, nbytes // 2, owner=alloc),
                                      device=device).view(torch.bfloat16)

    def __del__(self):
        # kernels already queued may still read or write the peers' buffers: unmap them only
        # once the device is idle (the own buffer goes with its last tensor view)
        try:
            torch.cuda.synchronize(self._device)
            for p in self._opened:
                _lib.load().dsv_peer_close(p)
            self.tensor = None
        except Exception:
            pass


class ScpPeerBuffers:
    """Selective KV gathering over NVLink for one rank of an SCP group (the g_s ranks holding
    the same heads; member g owns the tokens [g span, (g+1) span)). Full-length per-head
    buffers addressed by global token — K, V bf16 and dK, dV fp32 [hs, L, D] — are mapped
    into every member (CUDA IPC through libdsv). A member pulls the marked remote K/V rows
    straight from their owners' buffers (dsv_scp_pull, NVLink loads) and pushes the
    gradients of those rows into the owners' accumulators (dsv_scp_push, red.add over
    NVLink); device barriers order the phases. Counts stay on the device, so the step is
    graph-capturable (the all-to-all form in HybridExchange reads them back to size its
    collectives)."""

    def __init__(self, hs: int, seq_len: int, head_dim: int, d_lr: int, group, device):
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        n = hs * seq_len * head_dim
        nl = hs * seq_len * d_lr
        self.hs, self.L, self.D, self.r = hs, seq_len, head_dim, d_lr
        self.off = {"k": 0, "v": 2 * n, "dk": 4 * n, "dv": 8 * n, "klr": 12 * n,
                    "slots": 12 * n + 2 * nl}
        nbytes = 12 * n + 2 * nl + 4 * (self.world + 1) + 256
        self.peer = _PeerBuffer(nbytes, group, device)
        b = self.peer.tensor                                   # bf16 view of the whole buffer
        shape = (hs, seq_len, head_dim)
        self.k = b[0:n].view(shape)
        self.v = b[n:2 * n].view(shape)
        self.acc = b[2 * n:6 * n].view(torch.float32).view((2,) + shape)   # dK, dV fp32
        self.klr = b[6 * n:6 * n + nl].view(hs, seq_len, d_lr)            # K_lr, all keys
        ptrs = np.asarray(self.peer.ptrs, dtype=np.int64)
        dev = b.device
        # the peers' K_lr regions as tensors of this process (NVLink reads by torch copies)
        self.peer_klr = [self.klr if g == self.rank else
                         torch.as_tensor(_CudaArray(int(ptrs[g]) + self.off["klr"], nl),
                                         device=dev).view(torch.bfloat16).view(hs, seq_len, d_lr)
                         for g in range(self.world)]
        self.peer_tab = {name: torch.from_numpy(ptrs + off).to(dev)
                         for name, off in self.off.items()}
        so = self.off["slots"]
        self._slots_tab = self.peer_tab["slots"]
        self._my_slots = int(ptrs[self.rank]) + so
        self._epoch = self._my_slots + 4 * self.world
        self.pulled = torch.zeros((1,), dtype=torch.int64, device=dev)   # rows fetched (ledger)
        torch.cuda.synchronize(dev)
        dist.barrier(group)

    def barrier(self):
        _lib.call("dsv_peer_barrier", self._slots_tab.data_ptr(), self._my_slots, self._epoch,
                  self.world, self.rank, torch.cuda.current_stream(self.k.device).cuda_stream)

    def pull(self, mark, span0: int, span_len: int):
        st = torch.cuda.current_stream(self.k.device).cuda_stream
        _lib.call("dsv_scp_pull", mark.data_ptr(), self.hs, self.L, span0, span_len,
                  self.peer_tab["k"].data_ptr(), self.peer_tab["v"].data_ptr(), self.k.data_ptr(),
                  self.v.data_ptr(), self.D, self.pulled.data_ptr(), st)

    def push(self, mark, span0: int, span_len: int):
        st = torch.cuda.current_stream(self.k.device).cuda_stream
        _lib.call("dsv_scp_push", mark.data_ptr(), self.hs, self.L, span0, span_len,
                  self.peer_tab["dk"].data_ptr(), self.peer_tab["dv"].data_ptr(),
                  self.acc[0].data_ptr(), self.acc[1].data_ptr(), self.D, st)


class PeerExchange:
    """HCP exchange over NVLink peer memory (one process per GPU, B200 NVSwitch).

    Every rank owns one peer-mapped buffer (CUDA IPC) holding the regions the DSV layer reads
    and returns: Q, K, V, dO [heads, L, D] and Q_lr, K_lr [heads, L, r] for its
    heads, and O, dQ, dK, dV [H, L/N, D] for its tokens. A sender writes its rows
    straight into the owner's region (dsv_copy_jobs on peer pointers), so pack,
    transfer and unpack are one kernel per direction; a device barrier on both
    sides orders the writes (cpsim.py:125-161 and 284-299 phases, same bytes as
    the all-to-all form, recorded in the same ledger).

    The returned head-major/token-major tensors are views of the buffer and stay
    valid until the next exchange.
    """

    def __init__(self, n_heads: int, seq_len: int, head_dim: int, d_lr: int, assignment,
                 group=None, device=None, splits: int = 16, *, plan_only=None):
        """plan_only=(rank, world, buffer_ptrs): index/job planning without a process
        group or device memory (host tests drive the job tables through an emulator)."""
        if plan_only is None:
            self.group = group if group is not None else dist.group.WORLD
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.group = None
            self.rank, self.world = int(plan_only[0]), int(plan_only[1])
        if seq_len % self.world:
            raise ValueError("sequence length must divide the rank count")
        self.H, self.L, self.D, self.r = int(n_heads), int(seq_len), int(head_dim), int(d_lr)
        self.chunk = self.L // self.world
        self.assignment = np.asarray(assignment, dtype=np.int64)
        if self.assignment.shape != (self.H,) or self.assignment.min() < 0 or self.assignment.max() >= self.world:
            raise ValueError("assignment must map every head to a rank")
        if (self.D * 2) % 16 or (self.r * 2) % 16:
            raise ValueError("peer exchange needs head_dim and d_lr multiples of 8")
        self.heads_of = [np.nonzero(self.assignment == r)[0] for r in range(self.world)]
        self.my_heads = self.heads_of[self.rank]
        self.hi_of = np.zeros(self.H, dtype=np.int64)
        for hs in self.heads_of:
            self.hi_of[hs] = np.arange(len(hs))
        self.splits = int(os.environ.get("DSV_COPY_SPLITS", splits))
        self.ledger = Ledger()
        nh_max = max(len(h) for h in self.heads_of)
        big, small, back = nh_max * self.L * self.D, nh_max * self.L * self.r, self.H * self.chunk * self.D
        names = [("q", big), ("k", big), ("v", big), ("do", big), ("qlr", small), ("klr", small),
                 ("o", back), ("dq", back), ("dk", back), ("dv", back),
                 ("flags", 2 * (self.world + 1)),        # u32 [world] barrier slots + epoch
                 ("flags2", 2 * (self.world + 1))]       # a second set for the side stream
        self.off, tot = {}, 0
        for n, sz in names:
            self.off[n] = tot
            tot += -(-sz // 64) * 64                       # keep regions 128-byte aligned
        self.total_elems = tot
        self._tables = {}
        if plan_only is not None:
            self.buf, self.peer = None, None
            self.ptrs = np.asarray(plan_only[2], dtype=np.int64)
            return
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.peer = _PeerBuffer(2 * tot, self.group, dev)
        self.buf = self.peer.tensor
        self.ptrs = np.asarray(self.peer.ptrs, dtype=np.int64)
        # barrier slots: [world] u32 arrival epochs + one u32 epoch counter (device side); set 0
        # orders the compute stream, set 1 the side stream of the overlapped input exchange
        # (each set's barriers run in the same order on every rank)
        self._bars = []
        for name in ("flags", "flags2"):
            so = 2 * self.off[name]
            tab = torch.tensor([int(p) + so for p in self.ptrs], dtype=torch.int64, device=dev)
            mine = int(self.ptrs[self.rank]) + so
            self._bars.append((tab, mine, mine + 4 * self.world))
        torch.cuda.synchronize(dev)
        dist.barrier(self.group)
        self._step = 0

    def _barrier(self, which: int = 0):
        """Device barrier over the ranks' peer buffers on the current stream (slot set
        `which`)."""
        tab, mine, epoch = self._bars[which]
        _lib.call("dsv_peer_barrier", tab.data_ptr(), mine, epoch, self.world, self.rank,
                  torch.cuda.current_stream(self.buf.device).cuda_stream)

    # ------------------------------------------------------------------ views
    def region(self, name: str) -> torch.Tensor:
        nh = len(self.my_heads)
        o = self.off[name]
        if name in ("q", "k", "v", "do"):
            return self.buf[o: o + nh * self.L * self.D].view(nh, self.L, self.D)
        if name in ("qlr", "klr"):
            return self.buf[o: o + nh * self.L * self.r].view(nh, self.L, self.r)
        return self.buf[o: o + self.H * self.chunk * self.D].view(self.H, self.chunk, self.D)

    # ------------------------------------------------------------------ job tables
    def _table(self, key, build, stream=None):
        """Device job table cached by the pointers it encodes. Uploaded from pinned host
        memory (kept alive with the table), so a step can be captured in a CUDA graph.
        stream: the stream that will read the table (default: the current one); the upload
        is ordered on it and the allocator told, so an evicted table is not reused while
        that stream may still read it. A captured graph keeps using its tables' addresses, so
        the cache drops tables only after 64 distinct input-pointer sets (a double-buffered
        host pipeline uses a handful)."""
        t = self._tables.get(key)
        if t is None:
            if len(self._tables) >= 64:
                self._tables.clear()
            host = torch.from_numpy(build()).pin_memory()
            st = stream or torch.cuda.current_stream(self.buf.device)
            with torch.cuda.stream(st):
                dev = host.to(self.buf.device, non_blocking=True)
            dev.record_stream(st)
            t = (dev, host)
            self._tables[key] = t
        return t[0]

    def _head_jobs(self, named):
        """Flat per-head jobs: this rank's token chunk of head h of each tensor [H, L/N, D]
        -> the owner's region rows [hi, rank * L/N, :)."""
        H, L, D, chunk, me = self.H, self.L, self.D, self.chunk, self.rank
        h = np.arange(H, dtype=np.int64)
        dst_base = self.ptrs[self.assignment]
        jobs = []
        for name, t in named:
            j = np.empty((H, 6), dtype=np.int64)
            j[:, 0] = t.data_ptr() + h * chunk * D * 2
            j[:, 1] = dst_base + 2 * (self.off[name] + (self.hi_of * L + me * chunk) * D)
            j[:, 2] = j[:, 3] = chunk * D * 2
            j[:, 4] = 1
            j[:, 5] = chunk * D * 2
            jobs.append(j)
        return np.ascontiguousarray(np.concatenate(jobs))

    def _lowrank_jobs(self, p):
        """Rows of P [L/N, 2, H, r] -> the owners' Q_lr / K_lr regions (32-byte rows)."""
        H, L, r, chunk, me = self.H, self.L, self.r, self.chunk, self.rank
        h = np.arange(H, dtype=np.int64)
        dst_base = self.ptrs[self.assignment]
        jobs = []
        for side, name in ((0, "qlr"), (1, "klr")):
            j = np.empty((H, 6), dtype=np.int64)
            j[:, 0] = p.data_ptr() + 2 * (side * H + h) * r
            j[:, 1] = dst_base + 2 * (self.off[name] + (self.hi_of * L + me * chunk) * r)
            j[:, 2] = 2 * H * r * 2
            j[:, 3] = r * 2
            j[:, 4] = chunk
            j[:, 5] = r * 2
            jobs.append(j)
        return np.ascontiguousarray(np.concatenate(jobs))

    def _fwd_jobs(self, q, k, v, do, p):
        return np.ascontiguousarray(np.concatenate([
            self._head_jobs((("q", q), ("k", k), ("v", v), ("do", do))), self._lowrank_jobs(p)]))

    def _back_jobs(self, tensors, names=("o", "dq", "dk", "dv")):
        L, D, chunk = self.L, self.D, self.chunk
        hs = self.my_heads
        nh = len(hs)
        hi = np.repeat(np.arange(nh, dtype=np.int64), self.world)
        dst_r = np.tile(np.arange(self.world, dtype=np.int64), nh)
        dst_h = np.repeat(hs.astype(np.int64), self.world)
        jobs = []
        for name, t in zip(names, tensors):
            j = np.empty((nh * self.world, 6), dtype=np.int64)
            j[:, 0] = t.data_ptr() + 2 * (hi * L + dst_r * chunk) * D
            j[:, 1] = self.ptrs[dst_r] + 2 * (self.off[name] + dst_h * chunk * D)
            j[:, 2] = j[:, 3] = chunk * D * 2
            j[:, 4] = 1
            j[:, 5] = chunk * D * 2
            jobs.append(j)
        return np.ascontiguousarray(np.concatenate(jobs))

    def rows(self, name: str):
        """(tab int64 [my_heads * world], world, chunk): where row (local head hi, token t) of a
        [my_heads, L, D] result lands in its token owner's `name` region — the address table the
        fused epilogues (dsv_sparse_fwd o_tab, dsv_sparse_bwd dq_tab, dsv_f32_to_bf16_rows) store
        through, so the output redistribution needs no separate copy."""
        rt = self.__dict__.setdefault("_row_tabs", {})      # kept for the exchange's lifetime
        t = rt.get(name)
        if t is None:
            hs = self.my_heads.astype(np.int64)
            tab = (self.ptrs[None, :] + 2 * (self.off[name] + hs[:, None] * self.chunk * self.D)
                   ).reshape(-1)
            t = rt[name] = torch.from_numpy(np.ascontiguousarray(tab)).to(self.buf.device)
        return t, self.world, self.chunk

    def begin_tokens(self):
        """Fused output redistribution: the kernels about to run store into the token owners'
        regions (every rank is past the previous step: the to_heads barrier ordered that)."""

    def finish_tokens(self):
        """After the fused epilogues: a device barrier publishes the peer stores; returns the
        views O, dQ, dK, dV [H, L/N, D] of this rank's tokens."""
        self._barrier()
        self._account(("output_redistribute", self.D), ("hcp_bwd_out", 3 * self.D), to_heads=False)
        return tuple(self.region(n) for n in ("o", "dq", "dk", "dv"))

    def _host_table(self, key, build):
        t = self._tables.get(key)
        if t is None:
            if len(self._tables) >= 64:
                self._tables.clear()
            t = build()
            self._tables[key] = t
        return t

    def _run(self, table):
        from . import ops

        self._barrier()                      # owners are done reading the previous contents
        ops.copy_jobs(table, self.splits)
        self._barrier()                      # every writer is done: regions are complete

    # ------------------------------------------------------------------ exchanges
    def to_heads(self, q, k, v, do, p):
        """q, k, v, do [H, L/N, D] and P [L/N, 2 H r] (this rank's tokens) ->
        views Q, K, V, dO [my_heads, L, D], Q_lr, K_lr [my_heads, L, r]."""
        self._check_in(q, k, v, do, p)
        key = ("f",) + tuple(t.data_ptr() for t in (q, k, v, do, p))
        self._run(self._table(key, lambda: self._fwd_jobs(q, k, v, do, p)))
        self._account(("hcp_fwd", 3 * self.D + 2 * self.r), ("hcp_bwd_in", self.D), to_heads=True)
        return tuple(self.region(n) for n in ("q", "k", "v", "do", "qlr", "klr"))

    def to_heads_overlapped(self, q, k, v, do, p, side: torch.cuda.Stream):
        """to_heads with the bulk behind the compute: Q_lr / K_lr travel on the current stream
        (the selection needs only them); on `side`, Q, K, V go under the selection with a
        copy grid of about one 256-thread CTA per SM (8 K registers, which fit next to the
        one-CTA-per-SM selection kernel's 55 K), then dO — needed only by the backward —
        under the forward in 128-thread CTAs (4 K registers: what the persistent forward's
        800 x 72 leave). Returns the six views and two events: Q / K / V in place, dO in
        place."""
        from . import ops

        self._check_in(q, k, v, do, p)
        dev = self.buf.device
        cur = torch.cuda.current_stream(dev)
        key = ("fo",) + tuple(t.data_ptr() for t in (q, k, v, do, p))
        low = self._table(key + ("lr",), lambda: self._lowrank_jobs(p))
        qkv = self._table(key + ("qkv",), lambda: self._head_jobs((("q", q), ("k", k), ("v", v))),
                          stream=side)
        dsj = self._table(key + ("do",), lambda: self._head_jobs((("do", do),)), stream=side)
        self._barrier()                      # owners are done reading the previous contents
        ops.copy_jobs(low, self.splits)      # first, at full width: the selection waits on it
        side.wait_stream(cur)
        sm = torch.cuda.get_device_properties(dev).multi_processor_count
        with torch.cuda.stream(side):
            ops.copy_jobs(qkv, max(1, -(-sm // qkv.shape[0])))
            self._barrier(1)                 # every writer's Q / K / V rows are in place
            done_qkv = torch.cuda.Event()
            done_qkv.record(side)
            ops.copy_jobs(dsj, max(1, -(-sm // dsj.shape[0])), threads=128)
            self._barrier(1)                 # ... and dO
            done_do = torch.cuda.Event()
            done_do.record(side)
        self._barrier()                      # Q_lr / K_lr complete
        self._account(("hcp_fwd", 3 * self.D + 2 * self.r), ("hcp_bwd_in", self.D), to_heads=True)
        return tuple(self.region(n) for n in ("q", "k", "v", "do", "qlr", "klr")), (done_qkv, done_do)

    def _check_in(self, q, k, v, do, p):
        for t in (q, k, v, do, p):
            if not t.is_contiguous() or t.dtype != torch.bfloat16:
                raise ValueError("peer exchange expects contiguous bf16 tensors")
        if q.shape != (self.H, self.chunk, self.D) or p.shape != (self.chunk, 2 * self.H * self.r):
            raise ValueError("shape does not match the exchange plan")

    def to_tokens(self, o, dq, dk, dv):
        """o, dq, dk, dv [my_heads, L, D] -> views [H, L/N, D] on the token owners."""
        nh = len(self.my_heads)
        for t in (o, dq, dk, dv):
            if t.shape != (nh, self.L, self.D) or not t.is_contiguous() or t.dtype != torch.bfloat16:
                raise ValueError("peer exchange expects contiguous bf16 [my_heads, L, D]")
        key = ("b",) + tuple(t.data_ptr() for t in (o, dq, dk, dv))
        self._run(self._table(key, lambda: self._back_jobs((o, dq, dk, dv))))
        self._account(("output_redistribute", self.D), ("hcp_bwd_out", 3 * self.D), to_heads=False)
        return tuple(self.region(n) for n in ("o", "dq", "dk", "dv"))

    def _account(self, *phases, to_heads: bool):
        nh = len(self.my_heads)
        remote_heads_out = self.H - nh                 # my tokens of other ranks' heads
        remote_in = nh * (self.world - 1)              # my heads' tokens held elsewhere
        for phase, width in phases:
            row = self.chunk * width * 2
            if to_heads:
                self.ledger.add(phase, remote_heads_out * row, remote_in * row)
            else:
                self.ledger.add(phase, remote_in * row, remote_heads_out * row)


def plan_heads(sparsities, seq_len: int, head_dim: int, world: int, balanced: bool = True):
    """Head -> rank assignment: sparsity-aware `balance_heads` or the contiguous split."""
    if not balanced:
        return cpmodel.contiguous_heads(len(sparsities), world).assignment
    loads = cpmodel.head_loads(sparsities, seq_len, head_dim)
    return cpmodel.balance_heads(loads, world).assignment


def plan_heads_from_profile(profile, block: int, seq_len: int, head_dim: int, world: int,
                            balanced: bool = True):
    """Sparsity-aware head re-balancing from MEASURED sparsity: the EMA per head of one
    transformer block in a `profiler.SparsityProfile` (filled by `measure_block_sparsity`
    on the GPU, reference profiler.py:48-152) -> head loads (1 - s_h) S^2 d -> the
    `balance_heads` assignment (cpmodel.py:73-210). Returns (assignment, sparsities); pass
    the sparsities to HeadParallelDSV / HybridDSV / DSVAttentionLayer for the per-head k."""
    sp = np.asarray(profile.head_emas(block), dtype=np.float64)
    if sp.size == 0:
        raise ValueError(f"no sparsity measured for block {block}")
    return plan_heads(sp, seq_len, head_dim, world, balanced), sp


class HybridExchange:
    """Hybrid head x selective-sequence CP: g_h-way HCP inside each of g_s SCP groups
    (cpsim.py:125-161), then selective KV gathering between the g_s ranks that hold the
    same heads (cpsim.py:164-216), and the output redistribution (cpsim.py:284-299).

    Rank layout and placements follow `cpmodel.rank_layout` ("hcp-first": the g_h ranks
    of a group are consecutive, "scp-first": strided). Every rank calls the constructor
    (it creates the sub-groups collectively). Requests are per head: a rank asks the
    peer holding span(g') for the union of the key rows its span's queries selected
    inside span(g'), and the peer serves exactly those rows; the ledger records the
    reference's byte model (8 B per head list + 4 B per index, 2 x D x width per row).
    """

    def __init__(self, n_heads: int, seq_len: int, assignment, g_h: int, g_s: int,
                 placement: str = "hcp-first", group=None):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if g_h * g_s != self.world:
            raise ValueError("g_h * g_s must equal the number of ranks")
        if seq_len % self.world:
            raise ValueError("sequence length must divide the rank count")
        self.H, self.L, self.g_h, self.g_s = int(n_heads), int(seq_len), int(g_h), int(g_s)
        self.chunk = self.L // self.world
        self.layout = cpmodel.rank_layout(self.world, g_h, g_s, placement)
        self.pos, self.grp = self.layout[self.rank]
        self.assignment = np.asarray(assignment, dtype=np.int64)
        if self.assignment.shape != (self.H,) or self.assignment.min() < 0 or self.assignment.max() >= g_h:
            raise ValueError("assignment must map every head to a position in [0, g_h)")
        self.heads = np.nonzero(self.assignment == self.pos)[0]
        ranks_of_group = [sorted(r for r in range(self.world) if self.layout[r][1] == g) for g in range(g_s)]
        ranks_at_pos = [sorted(r for r in range(self.world) if self.layout[r][0] == p) for p in range(g_h)]
        glob = (lambda rs: rs) if group is None else (lambda rs: [dist.get_global_rank(group, r) for r in rs])
        hcp_groups = [dist.new_group(glob(rs)) for rs in ranks_of_group]
        scp_groups = [dist.new_group(glob(rs)) for rs in ranks_at_pos]
        self.hcp_group, self.scp_group = hcp_groups[self.grp], scp_groups[self.pos]
        self.spans = [np.sort(np.concatenate([np.arange(r * self.chunk, (r + 1) * self.chunk)
                                              for r in rs])) for rs in ranks_of_group]
        self.span = self.spans[self.grp]
        self.span_len = self.span.size
        self.span_of = np.empty(self.L, dtype=np.int64)       # global row -> SCP group
        self.local_at = np.empty(self.L, dtype=np.int64)      # global row -> index in its span
        for g, sp in enumerate(self.spans):
            self.span_of[sp] = g
            self.local_at[sp] = np.arange(sp.size)
        self.hcp = HeadParallelExchange(self.H, self.span_len, self.assignment, self.hcp_group)
        self.ledger = self.hcp.ledger                           # one ledger for all phases

    # ------------------------------------------------------------------ requests
    def requests_from_sets(self, sets):
        """sets: per head (global id) a list over the global queries of index arrays.
        Returns {peer group: [sorted unique int64 rows of span(peer), per local head]}."""
        req = {}
        for g in range(self.g_s):
            if g == self.grp:
                continue
            per_head = []
            for h in self.heads:
                need = np.unique(np.concatenate([np.asarray(sets[h][q], dtype=np.int64)
                                                 for q in self.span] or [np.zeros(0, np.int64)]))
                per_head.append(need[self.span_of[need] == g])
            req[g] = per_head
        return req

    def requests_from_idx(self, idx, counts):
        """GPU form: idx int32 [heads, groups, k_max] of global key rows (group r of head h
        valid up to counts[h, r]); same result as requests_from_sets."""
        hp = idx.shape[0]
        mark = torch.zeros((hp, self.L), dtype=torch.bool, device=idx.device)
        kmax = idx.shape[2]
        valid = torch.arange(kmax, device=idx.device)[None, None, :] < counts[:, :, None]
        for h in range(hp):
            rows = idx[h][valid[h]].long()
            mark[h, rows] = True
        span_of = torch.from_numpy(self.span_of).to(idx.device)
        req = {}
        for g in range(self.g_s):
            if g == self.grp:
                continue
            sel = mark & (span_of == g)[None, :]
            req[g] = [torch.nonzero(sel[h]).flatten().cpu().numpy() for h in range(hp)]
        return req

    # ------------------------------------------------------------------ exchanges
    def _a2a(self, send_parts, dtype, device, width):
        """all-to-all over the SCP group: send_parts[g] = tensor [n_g, width] to group g."""
        g_s = self.g_s
        cnt = torch.tensor([p.shape[0] for p in send_parts], dtype=torch.int64, device=device)
        rcnt = torch.empty_like(cnt)
        dist.all_to_all_single(rcnt, cnt, group=self.scp_group)
        rc = [int(x) for x in rcnt.cpu()]
        send = torch.cat([p.reshape(-1, width).to(dtype) for p in send_parts]) if sum(
            p.shape[0] for p in send_parts) else torch.zeros((0, width), dtype=dtype, device=device)
        recv = torch.empty((sum(rc), width), dtype=dtype, device=device)
        dist.all_to_all_single(recv, send, rc, [p.shape[0] for p in send_parts], group=self.scp_group)
        return list(torch.split(recv, rc)), rc

    def fetch_kv(self, k_span, v_span, req):
        """k_span, v_span [heads, span_len, D] (this rank's heads over its span).
        req: {peer group: [rows per head]} -> {peer group: (K rows, V rows) per head}."""
        dev, D = k_span.device, k_span.shape[2]
        hp = k_span.shape[0]          # this rank's sparse heads (dense ones take the ring)
        # 1. requested row lists (per head counts + ids) -> owners
        ids_parts, cnt_parts = [], []
        for g in range(self.g_s):
            per_head = req.get(g, [np.zeros(0, np.int64)] * hp)
            cnt_parts.append(torch.tensor([len(r) for r in per_head], dtype=torch.int64, device=dev)[:, None])
            ids_parts.append(torch.from_numpy(np.concatenate(per_head).astype(np.int64)
                                              if hp else np.zeros(0, np.int64)).to(dev)[:, None])
            if g != self.grp:
                n_idx = sum(len(r) for r in per_head)
                self.ledger.add("scp_index_exchange", 8 * hp + 4 * n_idx, 0)
        got_cnt, _ = self._a2a(cnt_parts, torch.int64, dev, 1)
        got_ids, _ = self._a2a(ids_parts, torch.int64, dev, 1)
        for g in range(self.g_s):
            if g != self.grp:
                self.ledger.add("scp_index_exchange", 0, 8 * hp + 4 * got_ids[g].shape[0])
        # 2. owners serve the rows: [K | V] per requested row, in request order
        local_at = torch.from_numpy(self.local_at).to(dev)
        serve, self._served = [], []
        for g in range(self.g_s):
            counts = [int(c) for c in got_cnt[g].flatten().cpu()]
            ids = got_ids[g].flatten()
            parts, o = [], 0
            for hi, c in enumerate(counts):
                at = local_at[ids[o:o + c]]
                parts.append(torch.cat([k_span[hi, at], v_span[hi, at]], dim=1))
                o += c
            self._served.append((counts, ids))
            rows = torch.cat(parts) if parts else torch.zeros((0, 2 * D), dtype=k_span.dtype, device=dev)
            serve.append(rows)
            if g != self.grp:
                self.ledger.add("scp_kv", rows.shape[0] * 2 * D * k_span.element_size(), 0)
        got_rows, _ = self._a2a(serve, k_span.dtype, dev, 2 * D)
        out = {}
        for g in range(self.g_s):
            if g == self.grp:
                continue
            per_head = req.get(g, [np.zeros(0, np.int64)] * hp)
            splits = [len(r) for r in per_head]
            rows = got_rows[g]
            self.ledger.add("scp_kv", 0, rows.shape[0] * 2 * D * k_span.element_size())
            out[g] = [(r[:, :D], r[:, D:]) for r in torch.split(rows, splits)]
        return out

    # ------------------------------------------------------------------ device-vectorised path
    def _dev_tables(self, device):
        key = ("dev", str(device))
        if getattr(self, "_dev_key", None) != key:
            self._span_of_d = torch.from_numpy(self.span_of).to(device)
            self._local_at_d = torch.from_numpy(self.local_at).to(device)
            self._span_d = torch.from_numpy(self.span).to(device)
            self._dev_key = key
        return self._span_of_d, self._local_at_d, self._span_d

    def requests_dev(self, mark):
        """mark: bool [heads, L], the global key rows this span's queries selected, per local
        head (any device). Returns (need, cnt): need int64 [n, 2] = (head, global row) of
        the remote rows, grouped by owner group, then head, then row; cnt int64 host
        [g_s, heads] = rows requested from each group per head. Same sets as
        requests_from_idx: the mark is regrouped as [owner group, head, span position] (one
        gather; a view when the spans are contiguous and in group order), so a single
        nonzero yields the rows already in request order."""
        dev = mark.device
        hp = mark.shape[0]
        key = ("perm", str(dev))
        if getattr(self, "_perm_key", None) != key:
            perm = np.concatenate(self.spans)
            self._perm_ident = bool(np.array_equal(perm, np.arange(self.L)))
            self._perm_d = torch.from_numpy(perm).to(dev)
            self._perm_key = key
        m = mark if self._perm_ident else mark.index_select(1, self._perm_d)
        mg = m.view(hp, self.g_s, self.span_len).transpose(0, 1).contiguous()   # [g_s, hp, span]
        mg[self.grp] = False                                                     # own span: local
        cnt = mg.sum(dim=2).cpu()                                                # [g_s, hp]
        nz = mg.nonzero()                                                        # (g, h, p) sorted
        rows = self._perm_d[nz[:, 0] * self.span_len + nz[:, 2]]
        need = torch.stack([nz[:, 1], rows], dim=1)
        return need, cnt

    def _a2a_fixed(self, send, recv_splits, send_splits):
        recv = torch.empty((sum(recv_splits),) + tuple(send.shape[1:]), dtype=send.dtype,
                           device=send.device)
        dist.all_to_all_single(recv, send.contiguous(), recv_splits, send_splits,
                               group=self.scp_group)
        return recv

    def fetch_kv_dev(self, k_span, v_span, need, cnt):
        """Device form of fetch_kv: k_span, v_span [heads, span_len, D]; (need, cnt) from
        requests_dev. Returns [n, 2 D] rows (K | V) aligned with `need`. Same bytes and
        ledger entries as fetch_kv (8 B per head list + 4 B per index; 2 D elements per row)."""
        dev, D = k_span.device, k_span.shape[2]
        hp = k_span.shape[0]
        _, local_at, _ = self._dev_tables(dev)
        g_s = self.g_s
        # 1. per-head counts, then the requested rows as indices inside the owner's span
        rcnt = torch.empty_like(cnt.to(dev))
        dist.all_to_all_single(rcnt, cnt.to(dev), group=self.scp_group)
        rcnt = rcnt.cpu()
        send_n = [int(cnt[g].sum()) for g in range(g_s)]
        recv_n = [int(rcnt[g].sum()) for g in range(g_s)]
        ids = local_at[need[:, 1]].to(torch.int32)
        got_ids = self._a2a_fixed(ids, recv_n, send_n)
        for g in range(g_s):
            if g != self.grp:
                self.ledger.add("scp_index_exchange", 8 * hp + 4 * send_n[g], 8 * hp + 4 * recv_n[g])
        # 2. owners serve [K | V] rows in request order (one gather per tensor)
        heads = torch.repeat_interleave(
            torch.arange(hp, device=dev).repeat(g_s), rcnt.flatten().to(dev),
            output_size=int(sum(recv_n)))
        flat = heads * self.span_len + got_ids.long()
        serve = torch.empty((flat.numel(), 2 * D), dtype=k_span.dtype, device=dev)
        if flat.numel():
            _gather_into(k_span.reshape(-1, D), flat, serve[:, :D])
            _gather_into(v_span.reshape(-1, D), flat, serve[:, D:])
        self._served_dev = (flat, recv_n)
        es = k_span.element_size()
        for g in range(g_s):
            if g != self.grp:
                self.ledger.add("scp_kv", recv_n[g] * 2 * D * es, send_n[g] * 2 * D * es)
        return self._a2a_fixed(serve, send_n, recv_n)

    def return_grads_dev(self, dk_full, dv_full, need, cnt, dk_span_flat_add):
        """Backward of fetch_kv_dev: gathers the fp32 gradients of the fetched rows from
        dk_full/dv_full [heads, L, D] (addressed by global row), sends them to the owners,
        which add them with dk_span_flat_add(rows_flat_in_span, dk_rows, dv_rows)."""
        dev, D = dk_full.device, dk_full.shape[2]
        g_s = self.g_s
        send_n = [int(cnt[g].sum()) for g in range(g_s)]
        flat_g = need[:, 0] * self.L + need[:, 1]
        rows = torch.empty((flat_g.numel(), 2 * D), dtype=dk_full.dtype, device=dev)
        if flat_g.numel():
            _gather_into(dk_full.reshape(-1, D), flat_g, rows[:, :D])
            _gather_into(dv_full.reshape(-1, D), flat_g, rows[:, D:])
        flat, recv_n = self._served_dev
        got = self._a2a_fixed(rows, recv_n, send_n)
        es = dk_full.element_size()
        for g in range(g_s):
            if g != self.grp:
                self.ledger.add("scp_grad", send_n[g] * 2 * D * es, recv_n[g] * 2 * D * es)
        if flat.numel():
            dk_span_flat_add(flat, got[:, :D], got[:, D:])

    def return_grads(self, dk_rows, dv_rows, dk_span, dv_span):
        """Backward of fetch_kv: dk_rows/dv_rows {peer group: [rows grads per head]} (fp32)
        are sent to the owners, which add them into dk_span/dv_span [heads, span_len, D]."""
        dev, D = dk_span.device, dk_span.shape[2]
        hp = dk_span.shape[0]
        parts = []
        for g in range(self.g_s):
            if g == self.grp or g not in dk_rows:
                parts.append(torch.zeros((0, 2 * D), dtype=dk_span.dtype, device=dev))
                continue
            parts.append(torch.cat([torch.cat([a, b], dim=1) for a, b in zip(dk_rows[g], dv_rows[g])])
                         if hp else torch.zeros((0, 2 * D), dtype=dk_span.dtype, device=dev))
            self.ledger.add("scp_grad", parts[-1].shape[0] * 2 * D * dk_span.element_size(), 0)
        got, _ = self._a2a(parts, dk_span.dtype, dev, 2 * D)
        local_at = torch.from_numpy(self.local_at).to(dev)
        for g in range(self.g_s):
            if g == self.grp:
                continue
            counts, ids = self._served[g]
            rows, o = got[g], 0
            self.ledger.add("scp_grad", 0, rows.shape[0] * 2 * D * dk_span.element_size())
            for hi, c in enumerate(counts):
                at = local_at[ids[o:o + c]]
                dk_span[hi].index_add_(0, at, rows[o:o + c, :D])
                dv_span[hi].index_add_(0, at, rows[o:o + c, D:])
                o += c


class _PhaseMarks:
    """Optional per-phase CUDA events on the compute stream (bench.py stage_ms)."""

    marks = None   # set to [] to record (name, cuda event) after each phase

    def _mark(self, name):
        if self.marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.marks.append((name, ev))

    def phase_ms(self):
        """Per-phase device time of the last step recorded with marks=[]."""
        torch.cuda.synchronize()
        m = self.marks or []
        return {b[0]: a[1].elapsed_time(b[1]) for a, b in zip(m, m[1:])}


class HeadParallelDSV(_PhaseMarks):
    """The DSV layer under HCP: sequence-sharded in, sequence-sharded out."""

    def __init__(self, grid, heads: int, head_dim: int, d_lr: int = 16, voxel=(8, 4, 4),
                 sparsity=0.9, balanced: bool = True, group=None, device="cuda",
                 transport: str = "auto", fused_out: bool | None = None):
        from .layer import DSVAttentionLayer

        self.world = dist.get_world_size(group)
        sp = np.broadcast_to(np.asarray(sparsity, dtype=np.float64), (heads,)).copy()
        self.assignment = plan_heads(sp, grid.size, head_dim, self.world, balanced)
        if np.bincount(self.assignment, minlength=self.world).min() == 0:
            # every rank sees the same plan, so all of them raise (no rank left in a collective);
            # cpmodel.solve_hybrid's rule: fewer heads than ranks needs g_s > 1 (HybridDSV)
            raise ValueError(f"head-parallel CP: {heads} heads leave a rank of {self.world} without "
                             "heads; use HybridDSV with g_s > 1")
        if transport == "auto":
            transport = "peer" if torch.device(device).type == "cuda" else "all_to_all"
        if transport not in ("peer", "all_to_all"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport
        # peer transport: the output redistribution rides on the kernels' epilogue stores
        # (DSV_FUSED_OUT=0 keeps the separate copy kernel for comparison)
        if fused_out is None:
            fused_out = os.environ.get("DSV_FUSED_OUT", "1") != "0"
        self.fused_out = bool(fused_out) and transport == "peer"
        if transport == "peer":
            self.ex = PeerExchange(heads, grid.size, head_dim, d_lr, self.assignment, group, device)
        else:
            self.ex = HeadParallelExchange(heads, grid.size, self.assignment, group)
        self.H, self.D, self.r = heads, head_dim, d_lr
        mine = self.ex.my_heads
        self.local = DSVAttentionLayer(grid, len(mine), head_dim, d_lr, voxel, sp[mine], device)
        # peer transport: Q / K / V / dO exchanged under the selection (DSV_OVERLAP_IN=0: after)
        self.overlap_in = transport == "peer" and os.environ.get("DSV_OVERLAP_IN", "1") != "0"
        self._side = torch.cuda.Stream(torch.device(device)) if self.overlap_in else None

    def step(self, x_local, wt, q, k, v, dout):
        """x_local [L/N, H*D]; q, k, v, dout [H, L/N, D] -> (out, dq, dk, dv) [H, L/N, D].

        transport "peer": two peer-memory copy kernels per step (inputs to the head
        owners, results back), outputs are views valid until the next step.
        transport "all_to_all": packed torch.distributed all-to-alls (any backend);
        the dO exchange runs asynchronously during the forward, and O travels back
        during the backward.
        """
        from . import ops

        if self.transport == "peer":
            return self._step_peer(x_local, wt, q, k, v, dout)
        H, r, D, ex = self.H, self.r, self.D, self.ex
        dev = q.device
        chunk = ex.chunk
        self._mark("start")
        p = ops.project(x_local, wt)                                   # [L/N, 2 H r]
        self._mark("project")
        hm = ex.send_rows_headmajor(dev)
        p_rows = p.view(chunk * 2 * H, r)
        fwd = ex.to_heads_packed([(q.reshape(H * chunk, D), hm), (k.reshape(H * chunk, D), hm),
                                  (v.reshape(H * chunk, D), hm),
                                  (p_rows, ex.send_rows_lowrank(0, dev)),
                                  (p_rows, ex.send_rows_lowrank(1, dev))], "hcp_fwd")
        h_do = ex.to_heads_packed([(dout.reshape(H * chunk, D), hm)], "hcp_bwd_in", async_op=True)
        self._mark("pack+send_fwd")
        ql, kl, vl, qlr, klr = ex.finish(fwd)
        self._mark("recv_fwd+unpack")
        sel = self.local.select_from_lowrank(qlr, klr)
        self._mark("select")
        out, lse = self.local.forward(ql, kl, vl, sel)
        self._mark("fwd")
        h_o = ex.to_tokens_packed([out], "output_redistribute", async_op=True)
        (dout_m,) = ex.finish(h_do)
        self._mark("send_o+recv_do")
        dq, dk, dv = self.local.backward(ql, kl, vl, out, lse, dout_m, sel)
        self._mark("bwd")
        grads = ex.finish(ex.to_tokens_packed([dq, dk, dv], "hcp_bwd_out"))
        self._mark("grads_back")
        (out_local,) = ex.finish(h_o)
        self._mark("o_back")
        return (out_local, *grads)

    def launches_per_step(self) -> int:
        """Kernels one peer-transport step launches: projection; barrier, one copy of all
        inputs, barrier (overlapped: barrier, Q_lr/K_lr copy, barrier, plus on the side stream
        the Q/K/V and dO copies with a barrier each); proxy gather; selection (fused: main +
        finish + list-mode re-run; unfused: scores GEMM + top-k); forward (+ list-mode re-run);
        backward (converting dK/dV in its tail, or two separate converts); then with fused
        outputs a barrier (else barrier + copy + barrier)."""
        n = 1 + 3 + (4 if self.overlap_in else 0) + 1 + (3 if self.local.fused_select() else 2)
        n += 2 + 1 + (0 if os.environ.get("DSV_BWD_CONVERT", "1") != "0" else 2)
        return n + (1 if self.fused_out else 3)

    def _step_peer(self, x_local, wt, q, k, v, dout):
        from . import ops

        loc = self.local
        self._mark("start")
        p = ops.project(x_local, wt)                                   # [L/N, 2 H r]
        self._mark("project")
        done_do = None
        if self.overlap_in:
            # Q / K / V travel on a side stream under the selection, dO under the forward
            (ql, kl, vl, dout_m, qlr, klr), (done_qkv, done_do) = self.ex.to_heads_overlapped(
                q, k, v, dout, p, self._side)
            self._mark("exchange_in")
            sel = loc.select_from_lowrank(qlr, klr)
            torch.cuda.current_stream(q.device).wait_event(done_qkv)
        else:
            ql, kl, vl, dout_m, qlr, klr = self.ex.to_heads(q, k, v, dout, p)
            self._mark("exchange_in")
            sel = loc.select_from_lowrank(qlr, klr)
        self._mark("select")
        ex = self.ex
        if self.fused_out:
            # output redistribution fused into the kernels: the forward epilogue also stores O
            # at the token owners, the backward's dQ epilogue and the dK / dV conversion store
            # there directly (NVLink peer stores), then one device barrier
            out, lse = loc.forward(ql, kl, vl, sel, out_rows=ex.rows("o"))
            self._mark("fwd")
            if done_do is not None:
                torch.cuda.current_stream(q.device).wait_event(done_do)
            loc.backward(ql, kl, vl, out, lse, dout_m, sel, dq_rows=ex.rows("dq"),
                         dkdv_rows=(ex.rows("dk"), ex.rows("dv")))
            self._mark("bwd")
            res = ex.finish_tokens()
            self._mark("exchange_out")
            return res
        out, lse = loc.forward(ql, kl, vl, sel)
        self._mark("fwd")
        if done_do is not None:
            torch.cuda.current_stream(q.device).wait_event(done_do)
        dq, dk, dv = loc.backward(ql, kl, vl, out, lse, dout_m, sel)
        self._mark("bwd")
        res = ex.to_tokens(out, dq, dk, dv)
        self._mark("exchange_out")
        return res


class HybridDSV(_PhaseMarks):
    """The DSV layer under hybrid CP (g_h x g_s, "hcp-first" placement).

    Each rank holds L/N tokens of all heads. Inside its SCP group (g_h consecutive
    ranks spanning L/g_s contiguous tokens) the inputs are resharded to the heads its
    position owns (packed all-to-all); K_lr is all-gathered between the g_s ranks with
    the same heads (r = 16 columns: the selection sees every key, as on one GPU); the
    voxel groups of the span are selected and their remote critical K/V rows gathered
    selectively (HybridExchange.fetch_kv); the attention runs on full-length buffers
    addressed by global token; the gradients of gathered rows go back to their owners
    and the outputs back to the token owners. The span must align with the voxel
    groups (L/g_s tokens = whole frames, a multiple of the voxel depth).

    Dense residual heads (`dense` mask, default: sparsity <= 0, i.e. the heads the
    dispatcher runs "full") skip selection and selective gathering: the g_s ranks that
    share such a head pass its K/V chunks around a ring (ring.RingKV, NCCL P2P) and merge
    the partial outputs by their LSE; the backward returns dK/dV with the ring.
    """

    def __init__(self, grid, heads: int, head_dim: int, d_lr: int, voxel, sparsity, g_h: int,
                 g_s: int, balanced: bool = True, group=None, device="cuda", dense=None,
                 transport: str = "auto", fused_out: bool | None = None):
        from .grouping import build_groups
        from .layer import DSVAttentionLayer
        from .ring import RingKV

        self.H, self.D, self.r, self.L = heads, head_dim, d_lr, grid.size
        sp = np.broadcast_to(np.asarray(sparsity, dtype=np.float64), (heads,)).copy()
        self.dense = (sp <= 0.0) if dense is None else np.broadcast_to(
            np.asarray(dense, dtype=bool), (heads,)).copy()
        self.sparsity = np.where(self.dense, 0.0, sp)
        self.assignment = plan_heads(self.sparsity, self.L, head_dim, g_h, balanced)
        self.ex = HybridExchange(heads, self.L, self.assignment, g_h, g_s, "hcp-first", group)
        span = self.ex.span
        self.s0, self.span_len = int(span[0]), int(span.size)
        if not np.array_equal(span, np.arange(self.s0, self.s0 + self.span_len)):
            raise ValueError("hybrid layer needs contiguous spans (hcp-first placement)")
        plan = build_groups(grid, voxel)
        inside = [i for i, m in enumerate(plan.members)
                  if m.min() >= self.s0 and m.max() < self.s0 + self.span_len]
        n_in = sum(plan.members[i].size for i in inside)
        if n_in != self.span_len:
            raise ValueError("the sequence span of an SCP group must hold whole voxel groups "
                             "(L / g_s tokens = a multiple of the voxel depth in frames)")
        self.heads = self.ex.heads
        self.device = torch.device(device)
        self.dloc = [i for i, h in enumerate(self.heads) if self.dense[h]]
        self.sloc = [i for i, h in enumerate(self.heads) if not self.dense[h]]
        self.local = (DSVAttentionLayer(grid, len(self.sloc), head_dim, d_lr, voxel,
                                        sp[self.heads[self.sloc]], device, groups=inside)
                      if self.sloc else None)
        self.ring = RingKV(self.ex.scp_group, ledger=self.ex.ledger) if self.dloc else None
        # the HCP leg inside each SCP group: NVLink peer-memory copy kernels on CUDA (as in
        # HeadParallelDSV), packed NCCL all-to-alls otherwise
        if transport == "auto":
            transport = "peer" if self.device.type == "cuda" else "all_to_all"
        self.peer = None
        if transport == "peer":
            self.peer = PeerExchange(heads, self.span_len, head_dim, d_lr, self.assignment,
                                     self.ex.hcp_group, self.device)
            self.peer.ledger = self.ex.ledger
        self._di = torch.tensor(self.dloc, dtype=torch.long, device=self.device)
        self._si = torch.tensor(self.sloc, dtype=torch.long, device=self.device)
        # selective KV over NVLink (one-sided pulls / pushes, device-side counts); the
        # all-to-all form (HybridExchange.fetch_kv_dev) stays for transport="all_to_all"
        self.scp = (ScpPeerBuffers(len(self.sloc), self.L, head_dim, d_lr, self.ex.scp_group,
                                   self.device)
                    if transport == "peer" and g_s > 1 and self.sloc else None)

    def work(self) -> dict:
        """Algorithmic work of this rank's heads over the whole sequence (sparse heads:
        the layer's per-head terms; dense heads: 4 L^2 D forward, 10 L^2 D backward)."""
        w = dict(self.local.work()) if self.local is not None else {
            "projection_flops": 0, "estimation_flops": 0, "topk_bytes": 0, "fwd_flops": 0,
            "bwd_flops": 0}
        nd = len(self.dloc)
        w["fwd_flops"] += 4 * nd * self.L * self.L * self.D
        w["bwd_flops"] += 10 * nd * self.L * self.L * self.D
        return w

    def _sparse(self, ql, kl, vl, dol, qlr, klr):
        """Selection + selective KV gathering + sparse attention for the sparse heads.
        Inputs [hs, span_len, .]; returns (out, dq, dk, dv) [hs, span_len, D] bf16."""
        from . import ops

        ex, L, r, D = self.ex, self.L, self.r, self.D
        hs, dev = ql.shape[0], ql.device
        sl = slice(self.s0, self.s0 + self.span_len)
        if self.scp is not None:
            return self._sparse_peer(ql, kl, vl, dol, qlr, klr)
        full = lambda t: torch.empty((hs, L, t.shape[2]), dtype=t.dtype, device=dev)
        Qf, Kf, Vf, dOf, Qlr = full(ql), full(kl), full(vl), full(dol), full(qlr)
        for dst, src in ((Qf, ql), (Kf, kl), (Vf, vl), (dOf, dol), (Qlr, qlr)):
            dst[:, sl] = src
        # every key's K_lr for the selection: all-gather over the ranks holding these heads
        parts = [torch.empty_like(klr) for _ in range(ex.g_s)]
        dist.all_gather(parts, klr.contiguous(), group=ex.scp_group)
        Klr = torch.cat([pp[:, None] for pp in parts], dim=1).reshape(hs, L, r)
        self._mark("exchange_in")
        sel = self.local.select_from_lowrank(Qlr, Klr)
        self._mark("select")
        if ex.g_s > 1:
            # the union of the span's critical keys per head, then the remote ones fetched
            mark = torch.zeros((hs, L), dtype=torch.bool, device=dev)
            ks = self.local.ks
            if len(set(ks)) == 1:      # one scatter over all heads (offset h * L)
                off = torch.arange(hs, device=dev, dtype=torch.int64)[:, None, None] * L
                mark.view(-1).index_fill_(0, (sel.idx[:, :, :ks[0]].long() + off).view(-1), True)
            else:
                for hi, kh in enumerate(ks):
                    mark[hi].index_fill_(0, sel.idx[hi, :, :kh].reshape(-1).long(), True)
            need, cnt = ex.requests_dev(mark)
            got = ex.fetch_kv_dev(kl, vl, need, cnt)
            flat = need[:, 0] * L + need[:, 1]
            Kf.view(-1, D).index_copy_(0, flat, got[:, :D])
            Vf.view(-1, D).index_copy_(0, flat, got[:, D:])
        self._mark("scp_fetch")
        out, lse = self.local.forward(Qf, Kf, Vf, sel, prepare_backward=False)
        self._mark("fwd")
        dk32 = torch.zeros((hs, L, D), dtype=torch.float32, device=dev)
        dv32 = torch.zeros_like(dk32)
        dq, dk32, dv32 = ops.sparse_bwd(Qf, Kf, Vf, out, dOf, lse, self.local.grp_rows,
                                        self.local.grp_size, sel.idx, sel.kcount,
                                        self.local.scale, dk32, dv32, tile_grp=self.local.tile_grp)
        self._mark("bwd")
        dk_span, dv_span = dk32[:, sl], dv32[:, sl]
        if ex.g_s > 1:
            def add_home(flat_span, dk_rows, dv_rows):     # rows addressed inside the span
                glob = (flat_span // self.span_len) * L + self.s0 + flat_span % self.span_len
                dk32.view(-1, D).index_add_(0, glob, dk_rows)
                dv32.view(-1, D).index_add_(0, glob, dv_rows)
            ex.return_grads_dev(dk32, dv32, need, cnt, add_home)
        dk = ops.f32_to_bf16(dk_span.contiguous())
        dv = ops.f32_to_bf16(dv_span.contiguous())
        self._mark("scp_grad")
        return out[:, sl].contiguous(), dq[:, sl].contiguous(), dk, dv

    def _sparse_peer(self, ql, kl, vl, dol, qlr, klr):
        """_sparse over NVLink peer memory: the span's K/V rows go into this rank's peer-mapped
        full-length buffers, the marked remote rows are pulled from their owners, the
        gradients of those rows pushed back into the owners' accumulators (dsv_scp_pull /
        dsv_scp_push between device barriers). No host synchronisation."""
        from . import ops

        ex, L, r, D, scp = self.ex, self.L, self.r, self.D, self.scp
        hs, dev = ql.shape[0], ql.device
        sl = slice(self.s0, self.s0 + self.span_len)
        Qf = torch.empty((hs, L, D), dtype=ql.dtype, device=dev)
        dOf = torch.empty_like(Qf)
        Qlr = torch.empty((hs, L, r), dtype=qlr.dtype, device=dev)
        Qf[:, sl], dOf[:, sl], Qlr[:, sl] = ql, dol, qlr
        scp.k[:, sl] = kl
        scp.v[:, sl] = vl
        scp.klr[:, sl] = klr
        scp.barrier()                       # every member's span rows are in place
        for g in range(ex.g_s):             # every key's K_lr for the selection (NVLink reads)
            if g != ex.grp:
                gs_ = slice(g * self.span_len, (g + 1) * self.span_len)
                scp.klr[:, gs_] = scp.peer_klr[g][:, gs_]
        Klr = scp.klr
        self._mark("exchange_in")
        sel = self.local.select_from_lowrank(Qlr, Klr)
        self._mark("select")
        mark = torch.zeros((hs, L), dtype=torch.bool, device=dev)
        ks = self.local.ks
        if len(set(ks)) == 1:
            off = torch.arange(hs, device=dev, dtype=torch.int64)[:, None, None] * L
            mark.view(-1).index_fill_(0, (sel.idx[:, :, :ks[0]].long() + off).view(-1), True)
        else:
            for hi, kh in enumerate(ks):
                mark[hi].index_fill_(0, sel.idx[hi, :, :kh].reshape(-1).long(), True)
        scp.pull(mark, self.s0, self.span_len)
        self._mark("scp_fetch")
        out, lse = self.local.forward(Qf, scp.k, scp.v, sel, prepare_backward=False)
        self._mark("fwd")
        scp.acc.zero_()
        dq, _, _ = ops.sparse_bwd(Qf, scp.k, scp.v, out, dOf, lse, self.local.grp_rows,
                                  self.local.grp_size, sel.idx, sel.kcount, self.local.scale,
                                  scp.acc[0], scp.acc[1], tile_grp=self.local.tile_grp)
        self._mark("bwd")
        scp.barrier()                       # every member's accumulators are zeroed and full
        scp.push(mark, self.s0, self.span_len)
        scp.barrier()                       # the remote gradients have landed
        dk = ops.f32_to_bf16(scp.acc[0][:, sl].contiguous())
        dv = ops.f32_to_bf16(scp.acc[1][:, sl].contiguous())
        self._mark("scp_grad")
        return out[:, sl].contiguous(), dq[:, sl].contiguous(), dk, dv

    def step(self, x_local, wt, q, k, v, dout):
        """x_local [L/N, H*D]; q, k, v, dout [H, L/N, D] -> (out, dq, dk, dv) [H, L/N, D]."""
        from . import ops

        hx = self.ex.hcp
        H, r, D = self.H, self.r, self.D
        hp, dev = len(self.heads), q.device
        chunk = hx.chunk
        self._mark("start")
        p = ops.project(x_local, wt)                                    # [L/N, 2 H r]
        self._mark("project")
        if self.peer is not None:
            ql, kl, vl, dol, qlr, klr = self.peer.to_heads(q, k, v, dout, p)
        else:
            hm = hx.send_rows_headmajor(dev)
            p_rows = p.view(chunk * 2 * H, r)
            h = hx.finish(hx.to_heads_packed(
                [(t.reshape(H * chunk, D), hm) for t in (q, k, v, dout)]
                + [(p_rows, hx.send_rows_lowrank(0, dev)), (p_rows, hx.send_rows_lowrank(1, dev))],
                "hcp_fwd"))
            ql, kl, vl, dol, qlr, klr = h
        if not self.dloc:
            o, dq, dk, dv = self._sparse(ql, kl, vl, dol, qlr, klr)
        else:
            o, dq, dk, dv = (torch.empty((hp, self.span_len, D), dtype=torch.bfloat16, device=dev)
                             for _ in range(4))
            if self.sloc:
                si = self._si
                res = self._sparse(ql[si], kl[si], vl[si], dol[si], qlr[si], klr[si])
                for dst, src in zip((o, dq, dk, dv), res):
                    dst[si] = src
            di = self._di
            qd, kd, vd, dod = ql[di], kl[di], vl[di], dol[di]
            od, lse = self.ring.forward(qd, kd, vd)
            self._mark("ring_fwd")
            res = (od, *self.ring.backward(qd, kd, vd, od, lse, dod))
            self._mark("ring_bwd")
            for dst, src in zip((o, dq, dk, dv), res):
                dst[di] = src
        if self.peer is not None:
            res = self.peer.to_tokens(o.contiguous(), dq.contiguous(), dk.contiguous(), dv.contiguous())
        else:
            h_o = hx.to_tokens_packed([o], "output_redistribute")
            grads = hx.finish(hx.to_tokens_packed([dq, dk, dv], "hcp_bwd_out"))
            res = (hx.finish(h_o)[0], *grads)
        self._mark("exchange_out")
        return res
