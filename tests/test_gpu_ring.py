"""Ring KV pass on one B200: the libdsv element kernels and the per-hop math.

* dsv_ring_lse_merge / dsv_ring_accum_bf16 / dsv_ring_accum_f32 against torch fp32/fp64
  formulas of the same contract (merge <= 1e-6, accumulations exact);
* a ring of n virtual ranks run hop by hop on one GPU (the schedule RingKV runs over NCCL;
  the schedule itself is checked on gloo in tests/test_ring_gloo.py): tcgen05 attention
  on each visiting chunk, LSE merge, dQ accumulation and traveling dK/dV accumulators,
  against the oracle's dense attention (full_attention semantics, attention.py:95-109) and
  its analytic gradients. Bars of the tcgen05 path (bf16 in, fp32 accumulate): O max-abs
  <= 3e-2 and rel-L2 <= 1.5e-2, LSE <= 2e-2, dQ/dK/dV rel-L2 <= 3e-2;
* RingKV with no process group (n = 1) is the dense tcgen05 attention.
"""

import math

import numpy as np
import pytest
import torch

import oracle
from paper_2502_07590_b200 import ops
from paper_2502_07590_b200.ring import RingKernels, RingKV

pytestmark = pytest.mark.gpu
LN2 = math.log(2.0)


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def test_ring_element_kernels(cuda):
    g = torch.Generator(device="cpu").manual_seed(3)
    H, L, D = 3, 200, 128
    acc = torch.randn((H, L, D), generator=g).to(cuda)
    part = torch.randn((H, L, D), generator=g).to(torch.bfloat16).to(cuda)
    la = (torch.randn((H, L), generator=g) * 4).to(cuda)
    lb = (torch.randn((H, L), generator=g) * 4).to(cuda)
    la[0, :5] = -float("inf")                               # one side saw no key
    lse_out = torch.empty_like(la)
    out = torch.empty((H, L, D), dtype=torch.bfloat16, device=cuda)
    a0 = acc.clone()
    ops.ring_lse_merge(acc, la, lse_out, part, lb, False, out)
    m = torch.maximum(la, lb)
    wa, wb = torch.exp2(la.double() - m.double()), torch.exp2(lb.double() - m.double())
    ref = (a0.double() * wa[..., None] + part.double() * wb[..., None]) / (wa + wb)[..., None]
    torch.testing.assert_close(acc.double(), ref, rtol=1e-5, atol=1e-6)
    torch.testing.assert_close(lse_out.double(), m.double() + torch.log2(wa + wb), rtol=1e-6, atol=1e-6)
    assert torch.equal(out, acc.to(torch.bfloat16))
    # first hop: plain copy
    ops.ring_lse_merge(acc, None, lse_out, part, lb, True)
    assert torch.equal(acc, part.float()) and torch.equal(lse_out, lb)
    # dQ accumulation
    x = torch.randn((H, L, D), generator=g).to(torch.bfloat16).to(cuda)
    a1 = acc.clone()
    ops.ring_accum_bf16(acc, x, False, out)
    assert torch.equal(acc, a1 + x.float()) and torch.equal(out, acc.to(torch.bfloat16))
    ops.ring_accum_bf16(acc, x, True)
    assert torch.equal(acc, x.float())
    # traveling accumulator
    p = torch.randn((2, H, L, D), generator=g).to(cuda)
    t = torch.randn((2, H, L, D), generator=g).to(cuda)
    t0, p0 = t.clone(), p.clone()
    ops.ring_accum_f32(t, p, False)
    assert torch.equal(t, t0 + p0) and not p.any()
    p.copy_(p0)
    ops.ring_accum_f32(t, p, True)
    assert torch.equal(t, p0) and not p.any()


@pytest.mark.parametrize("n,chunk,D", [(3, 384, 128), (4, 256, 64), (2, 1000, 128)])
def test_ring_hops_match_dense_oracle(cuda, n, chunk, D):
    H = 2
    L = n * chunk
    g = torch.Generator(device="cpu").manual_seed(11 + n)
    Q, Kf, V, dO = (torch.randn((H, L, D), generator=g).to(torch.bfloat16) for _ in range(4))
    Qd, Kd, Vd, dOd = (t.to(cuda) for t in (Q, Kf, V, dO))
    ch = lambda t, r: t[:, r * chunk:(r + 1) * chunk].contiguous()
    kern = RingKernels(chunk, chunk, H, D, device=cuda)
    outs, lses = [], []
    for p in range(n):                                       # forward, rank p
        acc = torch.empty((H, chunk, D), dtype=torch.float32, device=cuda)
        lse = [torch.empty((H, chunk), dtype=torch.float32, device=cuda) for _ in range(2)]
        out = torch.empty((H, chunk, D), dtype=torch.bfloat16, device=cuda)
        for t in range(n):
            j = (p - t) % n
            o_t, l_t = kern.attend(ch(Qd, p), ch(Kd, j), ch(Vd, j))
            kern.merge(acc, lse[(t - 1) % 2] if t else None, lse[t % 2], o_t, l_t, t == 0,
                       out if t == n - 1 else None)
        outs.append(out)
        lses.append(lse[(n - 1) % 2].clone())
    O = torch.cat(outs, dim=1)
    LSE = torch.cat(lses, dim=1)
    # backward: every rank's dQ, dK/dV accumulators per chunk (the ring delivers them home)
    dq = torch.empty_like(Qd)
    dkv = torch.zeros((n, 2, H, chunk, D), dtype=torch.float32, device=cuda)
    for p in range(n):
        part = torch.zeros((2, H, chunk, D), dtype=torch.float32, device=cuda)
        dq_acc = torch.empty((H, chunk, D), dtype=torch.float32, device=cuda)
        dq_p = torch.empty((H, chunk, D), dtype=torch.bfloat16, device=cuda)
        for t in range(n):
            j = (p - t) % n
            dq_t = kern.grad(ch(Qd, p), ch(Kd, j), ch(Vd, j), ch(O, p), ch(dOd, p),
                             ch(LSE, p), part[0], part[1])
            kern.accum_dq(dq_acc, dq_t, t == 0, dq_p if t == n - 1 else None)
            kern.accum_kv(dkv[j], part, False)
        dq[:, p * chunk:(p + 1) * chunk] = dq_p
    dK = torch.cat([dkv[j, 0] for j in range(n)], dim=1)
    dV = torch.cat([dkv[j, 1] for j in range(n)], dim=1)
    torch.cuda.synchronize()
    qn, kn, vn, don = (t.double().numpy() for t in (Q, Kf, V, dO))
    allk = [np.arange(L)]
    for h in range(H):
        ref, ref_lse = oracle.grouped_attention_fwd(qn[h], kn[h], vn[h], allk, allk)
        got = O[h].float().cpu().numpy()
        assert np.max(np.abs(got - ref)) <= 3e-2 and _rel(got, ref) <= 1.5e-2
        assert np.max(np.abs(LSE[h].cpu().numpy() * LN2 - ref_lse)) <= 2e-2
        rdq, rdk, rdv = oracle.grouped_attention_bwd(qn[h], kn[h], vn[h], allk, allk, don[h])
        assert _rel(dq[h].float().cpu().numpy(), rdq) <= 3e-2
        assert _rel(dK[h].cpu().numpy(), rdk) <= 3e-2
        assert _rel(dV[h].cpu().numpy(), rdv) <= 3e-2


def test_ring_single_rank_is_dense_attention(cuda):
    H, L, D = 2, 640, 128
    g = torch.Generator(device="cpu").manual_seed(5)
    Q, Kf, V, dO = (torch.randn((H, L, D), generator=g).to(torch.bfloat16) for _ in range(4))
    ring = RingKV()
    assert ring.n == 1
    Qd, Kd, Vd, dOd = (t.to(cuda) for t in (Q, Kf, V, dO))
    out, lse = ring.forward(Qd, Kd, Vd)
    dq, dk, dv = ring.backward(Qd, Kd, Vd, out, lse, dOd)
    torch.cuda.synchronize()
    assert torch.equal(Kd.cpu(), Kf) and torch.equal(Vd.cpu(), V)    # inputs untouched
    qn, kn, vn, don = (t.double().numpy() for t in (Q, Kf, V, dO))
    allk = [np.arange(L)]
    for h in range(H):
        ref, _ = oracle.grouped_attention_fwd(qn[h], kn[h], vn[h], allk, allk)
        assert np.max(np.abs(out[h].float().cpu().numpy() - ref)) <= 3e-2
        rdq, rdk, rdv = oracle.grouped_attention_bwd(qn[h], kn[h], vn[h], allk, allk, don[h])
        for got, r in ((dq, rdq), (dk, rdk), (dv, rdv)):
            assert _rel(got[h].float().cpu().numpy(), r) <= 3e-2
