"""Kernel-level parity on the GPU: libdsv (through its C ABI) vs the CPU oracle.

Tolerances (north_star: bit-exact selection, stated bf16/fp32 tolerance for
floating point):
  * top-k indices and thresholds: bit-exact (==) given identical fp32 scores;
  * tcgen05 GEMM (bf16 in, fp32 acc): |err| <= 2e-3 * sqrt(K) * max|ref| scale;
  * tensor-core sparse attention (bf16 in/out): max-abs <= 3e-2, rel-L2 <= 1.5e-2 for O;
    gradients rel-L2 <= 3e-2, against the fp64 oracle on the same bf16-rounded inputs;
  * CUDA-core CSR path (fp32 math): max-abs <= 2e-5.
"""

import math

import numpy as np
import pytest
import torch

import oracle
from paper_2502_07590_b200 import ops
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.grouping import build_groups

pytestmark = pytest.mark.gpu


def _rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


# ---------------------------------------------------------------- K2 top-k
def _check_topk(scores_np, ks, rows_per_head, cuda):
    s = torch.from_numpy(scores_np.astype(np.float32)).to(cuda)
    kp = torch.tensor(ks, dtype=torch.int32, device=cuda)
    idx, thr = ops.topk_rows(s, kp, rows_per_head)
    torch.cuda.synchronize()
    idx = idx.cpu().numpy()
    thr = thr.cpu().numpy()
    per_row_k = np.repeat(np.asarray(ks), rows_per_head)[: scores_np.shape[0]]
    ref_idx, ref_thr = oracle.topk_from_scores(scores_np.astype(np.float32), per_row_k)
    for r in range(scores_np.shape[0]):
        kr = per_row_k[r]
        np.testing.assert_array_equal(idx[r, :kr], ref_idx[r, :kr], err_msg=f"row {r} k={kr}")
    assert np.all(thr == ref_thr.astype(np.float32))


@pytest.mark.parametrize("L", [1, 7, 128, 1000, 4096, 32000])
def test_topk_random(cuda, L):
    rng = np.random.default_rng(L)
    R = 24
    scores = rng.standard_normal((R, L)).astype(np.float32)
    ks = [int(x) for x in rng.integers(1, L + 1, size=3)]
    _check_topk(scores, ks, R // 3, cuda)


def test_topk_unaligned_row_stride_many_rows(cuda):
    # row stride 4095 floats (rows not 16-byte aligned) and more rows than 2 x SMs, so the
    # kernel's look-ahead L2 prefetch would be issued (it must skip unaligned rows)
    rng = np.random.default_rng(4095)
    scores = rng.standard_normal((600, 4095)).astype(np.float32)
    _check_topk(scores, [409, 1, 4000], 200, cuda)


def test_topk_global_path(cuda):
    rng = np.random.default_rng(5)
    L = 70000  # beyond the shared-memory row budget
    scores = rng.standard_normal((4, L)).astype(np.float32)
    _check_topk(scores, [7000, 1], 2, cuda)


@pytest.mark.parametrize("L,ks", [(131072, [13108, 65536, 1, 131071]), (100003, [10001, 3])])
def test_topk_streaming_long_rows(cuda, L, ks):
    # rows beyond the shared-memory budget: two-pass streaming kernel (topk_stream.cu)
    rng = np.random.default_rng(L)
    scores = (rng.standard_normal((2 * len(ks), L)) * rng.uniform(0.1, 10, size=(2 * len(ks), 1))).astype(np.float32)
    _check_topk(scores, ks, 2, cuda)


def test_topk_streaming_c5_rows(cuda):
    # c5 row length (L = 524288, 32x128x128) at k = 52429 (90% sparsity) and the extremes
    rng = np.random.default_rng(524288)
    L = 524288
    scores = rng.standard_normal((6, L)).astype(np.float32)
    scores[4] = np.round(scores[4] * 4)        # heavy ties
    _check_topk(scores, [52429, 1, L - 1], 2, cuda)


def test_topk_streaming_ties_zero_inf(cuda):
    rng = np.random.default_rng(9)
    L = 90000
    ints = rng.integers(-3, 4, size=(4, L)).astype(np.float32)
    vals = np.array([-0.0, 0.0, 1.0, -1.0, np.inf, -np.inf, 0.5], dtype=np.float32)
    special = vals[rng.integers(0, vals.size, size=(4, L))]
    _check_topk(np.concatenate([ints, special]), [1, 9000, 45000, 89999], 2, cuda)


def test_topk_ties_integer_scores(cuda):
    rng = np.random.default_rng(1)
    L = 5000
    scores = rng.integers(-3, 4, size=(16, L)).astype(np.float32)
    _check_topk(scores, [1, 500, 2500, 4999], 4, cuda)


def test_topk_all_equal_takes_lowest(cuda):
    scores = np.ones((3, 1000), dtype=np.float32)
    s = torch.from_numpy(scores).to(cuda)
    idx, thr = ops.topk_rows(s, torch.tensor([37], dtype=torch.int32, device=cuda), 3)
    assert np.array_equal(idx.cpu().numpy(), np.tile(np.arange(37), (3, 1)))
    assert np.all(thr.cpu().numpy() == 1.0)


def test_topk_signed_zero_and_inf(cuda):
    rng = np.random.default_rng(2)
    vals = np.array([-0.0, 0.0, 1.0, -1.0, np.inf, -np.inf], dtype=np.float32)
    scores = vals[rng.integers(0, vals.size, size=(8, 3000))]
    _check_topk(scores, [1, 10, 1500, 2999], 2, cuda)


def test_topk_scores_from_lowrank_product(cuda):
    # the K1b -> K2 chain: fp32 SIMT scores, then selection, vs oracle on the same scores
    rng = np.random.default_rng(3)
    q = rng.standard_normal((2, 64, 16)).astype(np.float32)
    k = rng.standard_normal((2, 4096, 16)).astype(np.float32)
    sc = ops.scores_f32(torch.from_numpy(q).to(cuda), torch.from_numpy(k).to(cuda))
    torch.cuda.synchronize()
    sc_np = sc.cpu().numpy()
    ref = np.einsum("hrt,hlt->hrl", q.astype(np.float64), k.astype(np.float64))
    assert np.max(np.abs(sc_np - ref)) < 1e-4
    _check_topk(sc_np.reshape(128, 4096), [410, 50], 64, cuda)


# ---------------------------------------------------------------- K1 GEMM
@pytest.mark.parametrize("M,N,K,nb", [(300, 768, 3072, 1), (260, 1000, 16, 3), (128, 128, 64, 1),
                                      (37, 200, 104, 2)])
def test_gemm_bf16(cuda, M, N, K, nb):
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    a = torch.randn((nb, M, K), generator=g).to(torch.bfloat16)
    b = torch.randn((nb, N, K), generator=g).to(torch.bfloat16)
    ref = torch.einsum("bmk,bnk->bmn", a.double(), b.double())
    c32 = ops.gemm_bf16(a.to(cuda), b.to(cuda), torch.float32).double().cpu()
    tol = 1e-4 * math.sqrt(K) * 4
    assert torch.max(torch.abs(c32 - ref)).item() < tol + 1e-3
    c16 = ops.gemm_bf16(a.to(cuda), b.to(cuda), torch.bfloat16).double().cpu()
    assert torch.max(torch.abs(c16 - ref) / (ref.abs() + 1.0)).item() < 1e-2


def test_project_matches_matmul(cuda):
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn((1000, 512), generator=g).to(torch.bfloat16)
    wt = (torch.randn((256, 512), generator=g) / math.sqrt(512)).to(torch.bfloat16)
    out = ops.project(x.to(cuda), wt.to(cuda)).double().cpu()
    ref = x.double() @ wt.double().T
    assert torch.max(torch.abs(out - ref)).item() < 2e-2


# ---------------------------------------------------------------- K3 attention
def _grouped_case(D, H, grid, voxel, ks, seed):
    rng = np.random.default_rng(seed)
    plan = build_groups(TokenGrid(*grid), voxel)
    L = plan.grid.size
    q = rng.standard_normal((H, L, D)).astype(np.float32)
    k = rng.standard_normal((H, L, D)).astype(np.float32)
    v = rng.standard_normal((H, L, D)).astype(np.float32)
    do = rng.standard_normal((H, L, D)).astype(np.float32)
    G = plan.n_groups
    kmax = max(ks)
    idx = np.zeros((H, G, kmax), dtype=np.int32)
    sets = []
    for h in range(H):
        per = []
        for g in range(G):
            sel = np.sort(rng.choice(L, size=ks[h], replace=False))
            idx[h, g, : ks[h]] = sel
            per.append(sel)
        sets.append(per)
    return plan, q, k, v, do, idx, sets


def _bf(x):
    return torch.from_numpy(x).to(torch.bfloat16)


@pytest.mark.parametrize("D", [128, 64])
def test_sparse_fwd_bwd_tc(cuda, D):
    H = 2
    plan, q, k, v, do, idx, sets = _grouped_case(D, H, (4, 8, 10), (4, 4, 8), [130, 257], seed=D)
    qb, kb, vb, dob = (_bf(t) for t in (q, k, v, do))
    rows, size = plan.tables(cuda)
    kcount = torch.tensor([130, 257], dtype=torch.int32, device=cuda)
    idx_t = torch.from_numpy(idx).to(cuda)
    out, lse = ops.sparse_fwd(qb.to(cuda), kb.to(cuda), vb.to(cuda), rows, size, idx_t, kcount)
    torch.cuda.synchronize()
    out = out.float().cpu().numpy()
    lse = lse.cpu().numpy()
    qd, kd, vd, dod = (t.double().numpy() for t in (qb, kb, vb, dob))
    for h in range(H):
        ref, ref_lse = oracle.grouped_attention_fwd(qd[h], kd[h], vd[h], plan.members, sets[h])
        assert np.max(np.abs(out[h] - ref)) < 3e-2, f"head {h}"
        assert _rel_l2(out[h], ref) < 1.5e-2
        assert np.max(np.abs(lse[h] * math.log(2.0) - ref_lse)) < 2e-2
    # backward with the kernel's own O / LSE
    out2, lse2 = ops.sparse_fwd(qb.to(cuda), kb.to(cuda), vb.to(cuda), rows, size, idx_t, kcount)
    dq, dk, dv = ops.sparse_bwd(qb.to(cuda), kb.to(cuda), vb.to(cuda), out2, dob.to(cuda), lse2,
                                rows, size, idx_t, kcount)
    torch.cuda.synchronize()
    dq, dk, dv = dq.float().cpu().numpy(), dk.cpu().numpy(), dv.cpu().numpy()
    for h in range(H):
        rdq, rdk, rdv = oracle.grouped_attention_bwd(qd[h], kd[h], vd[h], plan.members, sets[h], dod[h])
        assert _rel_l2(dq[h], rdq) < 3e-2, f"dq head {h}: {_rel_l2(dq[h], rdq)}"
        assert _rel_l2(dk[h], rdk) < 3e-2, f"dk head {h}: {_rel_l2(dk[h], rdk)}"
        assert _rel_l2(dv[h], rdv) < 3e-2, f"dv head {h}: {_rel_l2(dv[h], rdv)}"


def test_sparse_fwd_full_set_equals_dense(cuda):
    D, H = 128, 1
    plan = build_groups(TokenGrid(2, 8, 16), (2, 8, 8))
    L = plan.grid.size
    rng = np.random.default_rng(9)
    q, k, v = (rng.standard_normal((H, L, D)).astype(np.float32) for _ in range(3))
    idx = np.tile(np.arange(L, dtype=np.int32), (H, plan.n_groups, 1))
    rows, size = plan.tables(cuda)
    out, _ = ops.sparse_fwd(_bf(q).to(cuda), _bf(k).to(cuda), _bf(v).to(cuda), rows, size,
                            torch.from_numpy(idx).to(cuda),
                            torch.tensor([L], dtype=torch.int32, device=cuda))
    ref = oracle.full_attention(*(_bf(t).double().numpy()[0] for t in (q, k, v)))
    assert np.max(np.abs(out.float().cpu().numpy()[0] - ref)) < 3e-2


@pytest.mark.parametrize("gain,where", [(1.0, "last"), (6.0, "last"), (6.0, "middle")])
def test_sparse_fwd_late_max_jump_on_some_rows(cuda, gain, where):
    # a few query rows meet a key in a later key block whose logit is far above the rows'
    # running max (online-softmax rescale), the other rows of the same warp do not: the
    # rescale must stay warp-uniform (tcgen05.ld/st are warp-collective). gain 1: a jump
    # of ~16 (log2) that the lazy-max pass absorbs; gain 6: ~98, beyond its 2^64 headroom,
    # so the tile is flagged and re-run with the per-block max exchange.
    D, H = 128, 1
    plan = build_groups(TokenGrid(4, 8, 16), (2, 8, 8))
    L = plan.grid.size
    rng = np.random.default_rng(11)
    q, k, v, do = (rng.standard_normal((H, L, D)).astype(np.float32) for _ in range(4))
    hot = rng.choice(L, size=20, replace=False)
    for i, r in enumerate(hot):
        k[0, (L - 1 - i) if where == "last" else (L // 2 + 3 * i)] = gain * q[0, r]
    idx = np.tile(np.arange(L, dtype=np.int32), (H, plan.n_groups, 1))
    rows, size = plan.tables(cuda)
    kc = torch.tensor([L], dtype=torch.int32, device=cuda)
    qb, kb, vb, dob = (_bf(t).to(cuda) for t in (q, k, v, do))
    idx_t = torch.from_numpy(idx).to(cuda)
    out, lse = ops.sparse_fwd(qb, kb, vb, rows, size, idx_t, kc)
    dq, dk, dv = ops.sparse_bwd(qb, kb, vb, out, dob, lse, rows, size, idx_t, kc)
    torch.cuda.synchronize()
    qd, kd, vd, dod = (_bf(t).double().numpy()[0] for t in (q, k, v, do))
    sets = [np.arange(L)] * plan.n_groups
    ref, ref_lse = oracle.grouped_attention_fwd(qd, kd, vd, plan.members, sets)
    assert np.max(np.abs(out.float().cpu().numpy()[0] - ref)) < 3e-2
    assert np.max(np.abs(lse.cpu().numpy()[0] * math.log(2.0) - ref_lse)) < 2e-2
    rdq, rdk, rdv = oracle.grouped_attention_bwd(qd, kd, vd, plan.members, sets, dod)
    assert _rel_l2(dq.float().cpu().numpy()[0], rdq) < 3e-2
    assert _rel_l2(dk.cpu().numpy()[0], rdk) < 3e-2
    assert _rel_l2(dv.cpu().numpy()[0], rdv) < 3e-2


# ---------------------------------------------------------------- CSR path
@pytest.mark.parametrize("D", [4, 64, 100])
def test_rows_fwd_bwd(cuda, D):
    rng = np.random.default_rng(D)
    H, L = 2, 50
    q, k, v, do = (rng.standard_normal((H, L, D)).astype(np.float32) for _ in range(4))
    lists = [[np.sort(rng.choice(L, size=int(rng.integers(1, L + 1)), replace=False))
              for _ in range(L)] for _ in range(H)]
    ptr = np.zeros(H * L + 1, dtype=np.int64)
    cols = np.concatenate([x for per in lists for x in per]).astype(np.int32)
    ptr[1:] = np.cumsum([x.size for per in lists for x in per])
    tq, tk, tv, tdo = (torch.from_numpy(t).to(cuda) for t in (q, k, v, do))
    tp, tc = torch.from_numpy(ptr).to(cuda), torch.from_numpy(cols).to(cuda)
    out, lse = ops.rows_fwd(tq, tk, tv, tp, tc)
    dq, dk, dv = ops.rows_bwd(tq, tk, tv, out, lse, tdo, tp, tc)
    torch.cuda.synchronize()
    for h in range(H):
        ref, ref_lse = oracle.rows_attention_fwd(q[h], k[h], v[h], lists[h])
        assert np.max(np.abs(out[h].cpu().numpy() - ref)) < 2e-5
        assert np.max(np.abs(lse[h].cpu().numpy() - ref_lse)) < 2e-5
        rdq, rdk, rdv = oracle.rows_attention_bwd(q[h], k[h], v[h], lists[h], do[h])
        assert np.max(np.abs(dq[h].cpu().numpy() - rdq)) < 1e-4
        assert np.max(np.abs(dk[h].cpu().numpy() - rdk)) < 1e-4
        assert np.max(np.abs(dv[h].cpu().numpy() - rdv)) < 1e-4


def test_sparse_fwd_deterministic_repeated(cuda):
    # the forward has no atomics: repeated launches on the same inputs must agree bit for
    # bit (a TMEM read/write race between the softmax warps shows up here first)
    D, H, k = 128, 4, 1024
    plan = build_groups(TokenGrid(16, 16, 32), (8, 4, 4))
    L, G = plan.grid.size, plan.n_groups
    g = torch.Generator(device="cpu").manual_seed(21)
    idx = torch.stack([torch.randperm(L, generator=g)[:k].sort().values for _ in range(H * G)])
    idx = idx.to(torch.int32).reshape(H, G, k).to(cuda)
    q, kk, v = (torch.randn((H, L, D), generator=g).to(torch.bfloat16).to(cuda) for _ in range(3))
    rows, size = plan.tables(cuda)
    kc = torch.full((H,), k, dtype=torch.int32, device=cuda)
    out0, lse0 = ops.sparse_fwd(q, kk, v, rows, size, idx, kc)
    for _ in range(8):
        out, lse = ops.sparse_fwd(q, kk, v, rows, size, idx, kc)
        assert torch.equal(out, out0) and torch.equal(lse, lse0)


def test_layer_backward_accumulators_zeroed_by_forward_or_itself(cuda):
    # the forward kernel zeroes the layer's dK/dV accumulators for the next backward; a
    # second backward (no forward in between) must zero them itself, and explicit
    # caller accumulators give the same gradients
    from paper_2502_07590_b200.layer import DSVAttentionLayer

    grid = TokenGrid(8, 16, 16)
    H, D = 3, 128
    layer = DSVAttentionLayer(grid, H, D, 16, (8, 4, 4), [0.5, 0.8, 0.9], cuda)
    L = grid.size
    g = torch.Generator(device="cpu").manual_seed(17)
    x = torch.randn((L, H * D), generator=g).to(torch.bfloat16).to(cuda)
    q, k, v, do = (torch.randn((H, L, D), generator=g).to(torch.bfloat16).to(cuda) for _ in range(4))
    sel = layer.select(x, layer.predictor_weights(seed=2))
    out, lse = layer.forward(q, k, v, sel)
    a = layer.backward(q, k, v, out, lse, do, sel)
    b = layer.backward(q, k, v, out, lse, do, sel)              # no forward in between
    dk_acc = torch.full((H, L, D), 7.0, device=cuda)             # garbage: must be zeroed
    dv_acc = torch.full((H, L, D), -3.0, device=cuda)
    c = layer.backward(q, k, v, out, lse, do, sel, dk_acc, dv_acc)
    torch.cuda.synchronize()
    for x1, x2, x3 in zip(a, b, c):
        assert _rel_l2(x2.float().cpu().numpy(), x1.float().cpu().numpy()) < 1e-3
        assert _rel_l2(x3.float().cpu().numpy(), x1.float().cpu().numpy()) < 1e-3


@pytest.mark.parametrize("D", [128, 64])
def test_backward_tail_conversion_equals_separate_pass(cuda, D):
    # the backward's tail conversion (dsv_sparse_bwd_convert: per-head completion counters,
    # CTAs out of tiles convert finished heads) must give the bits of the separate fp32 ->
    # bf16 pass over the same accumulators — at 512 tiles on 148 persistent CTAs, so heads
    # finish while other CTAs are still on earlier ones
    H, k = 4, 1024
    plan = build_groups(TokenGrid(16, 16, 32), (8, 4, 4))
    L, G = plan.grid.size, plan.n_groups
    g = torch.Generator(device="cpu").manual_seed(33 + D)
    idx = torch.stack([torch.randperm(L, generator=g)[:k].sort().values for _ in range(H * G)])
    idx = idx.to(torch.int32).reshape(H, G, k).to(cuda)
    q, kk, v, do = (torch.randn((H, L, D), generator=g).to(torch.bfloat16).to(cuda) for _ in range(4))
    rows, size = plan.tables(cuda)
    kc = torch.full((H,), k, dtype=torch.int32, device=cuda)
    out, lse = ops.sparse_fwd(q, kk, v, rows, size, idx, kc)
    dkdv = torch.empty((2, H, L, D), device=cuda, dtype=torch.bfloat16)
    dq1, dk32, dv32 = ops.sparse_bwd(q, kk, v, out, do, lse, rows, size, idx, kc, dkdv_out=dkdv)
    torch.cuda.synchronize()
    assert torch.equal(dkdv[0], ops.f32_to_bf16(dk32)) and torch.equal(dkdv[1], ops.f32_to_bf16(dv32))
    dq2, _, _ = ops.sparse_bwd(q, kk, v, out, do, lse, rows, size, idx, kc)
    assert torch.equal(dq1, dq2)
