"""Ring KV pass (paper_2502_07590_b200.ring.RingKV) on gloo, world sizes 2 and 3 (CPU).

The ring schedule, the neighbour transfers, the LSE merge order and the traveling dK/dV
accumulators are the code the NCCL path runs; the per-hop device work is replaced by a
float64 torch stand-in that honours the libdsv contract (partial rows normalised by their
own sum, LSE in log2, dK/dV parts accumulated in place, parts re-zeroed by accum_kv).
Checked against the oracle's dense attention (full_attention semantics, attention.py:95-109)
and its analytic gradients over the concatenated sequence, plus the per-phase byte ledger.
"""

import math
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

LN2 = math.log(2.0)


class CpuKernels:
    """float64 stand-in for ring.RingKernels (same argument contract)."""

    def __init__(self, scale):
        self.scale = scale

    def attend(self, q, k, v):
        s = torch.einsum("hqd,hkd->hqk", q, k) * self.scale
        lse = torch.logsumexp(s, dim=-1)
        return torch.einsum("hqk,hkd->hqd", torch.softmax(s, -1), v), lse / LN2

    def grad(self, q, k, v, out, dout, lse, dk_part, dv_part):
        s = torch.einsum("hqd,hkd->hqk", q, k) * self.scale
        p = torch.exp(s - lse[..., None] * LN2)
        dp = torch.einsum("hqd,hkd->hqk", dout, v)
        delta = (dout * out).sum(-1, keepdim=True)
        ds = p * (dp - delta) * self.scale
        dk_part += torch.einsum("hqk,hqd->hkd", ds, q)
        dv_part += torch.einsum("hqk,hqd->hkd", p, dout)
        return torch.einsum("hqk,hkd->hqd", ds, k)

    @staticmethod
    def merge(acc, lse_in, lse_out, part, lse_part, first, out=None):
        if first:
            acc.copy_(part)
            lse_out.copy_(lse_part)
        else:
            m = torch.maximum(lse_in, lse_part)
            wa, wb = torch.exp2(lse_in - m), torch.exp2(lse_part - m)
            acc.copy_((acc * wa[..., None] + part * wb[..., None]) / (wa + wb)[..., None])
            lse_out.copy_(m + torch.log2(wa + wb))
        if out is not None:
            out.copy_(acc)

    @staticmethod
    def accum_dq(acc, x, first, out=None):
        acc.copy_(x if first else acc + x)
        if out is not None:
            out.copy_(acc)

    @staticmethod
    def accum_kv(acc, part, first):
        acc.copy_(part if first else acc + part)
        part.zero_()

    @staticmethod
    def to_bf16(x):
        return x.clone()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2502_07590_b200.cp import Ledger
        from paper_2502_07590_b200.ring import RingKV

        H, chunk, D = 2, 24, 16
        L = chunk * world
        rng = np.random.default_rng(5)
        Q, Kf, V, dO = (rng.standard_normal((H, L, D)) for _ in range(4))
        sl = slice(rank * chunk, (rank + 1) * chunk)
        loc = [torch.from_numpy(t[:, sl].copy()) for t in (Q, Kf, V, dO)]
        ledger = Ledger()
        ring = RingKV(kernels=CpuKernels(1.0 / math.sqrt(D)), ledger=ledger)
        out, lse = ring.forward(*loc[:3])
        dq, dk, dv = ring.backward(*loc[:3], out, lse, loc[3])
        for t, full in zip(loc, (Q, Kf, V, dO)):          # inputs are never mutated
            np.testing.assert_array_equal(t.numpy(), full[:, sl])
        everything = [np.arange(L)]   # accumulators are fp32 (the product's), hence 2e-6
        for h in range(H):
            ref, ref_lse = oracle.grouped_attention_fwd(Q[h], Kf[h], V[h], [np.arange(L)], everything)
            np.testing.assert_allclose(out[h].numpy(), ref[sl], atol=2e-6)
            np.testing.assert_allclose(lse[h].numpy() * LN2, ref_lse[sl], atol=2e-6)
            rdq, rdk, rdv = oracle.grouped_attention_bwd(Q[h], Kf[h], V[h], [np.arange(L)], everything, dO[h])
            np.testing.assert_allclose(dq[h].numpy(), rdq[sl], atol=2e-6)
            np.testing.assert_allclose(dk[h].numpy(), rdk[sl], atol=2e-6)
            np.testing.assert_allclose(dv[h].numpy(), rdv[sl], atol=2e-6)
        exp = ring.expected_bytes(H, chunk, D, elem=8)   # fp64 K/V payloads, fp32 accumulators
        assert ledger.sent["ring_kv"] == exp["ring_kv"] == ledger.received["ring_kv"]
        assert ledger.sent["ring_kv_bwd"] == exp["ring_kv_bwd"]
        assert ledger.sent["ring_grad"] == exp["ring_grad"] == ledger.received["ring_grad"]
        q.put((rank, "ok"))
    except Exception as e:  # surface worker failures to the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert results == {r: "ok" for r in range(world)}, results
    assert all(p.exitcode == 0 for p in procs)


def test_ring_kv_gloo_world2():
    _run(2)


def test_ring_kv_gloo_world3():
    _run(3)
