"""Fused K1b + K2 (select_fused.cu) against the unfused path (tcgen05 GEMM scores + K2
top-k, itself pinned to the oracle in test_gpu_kernels.py) and against the oracle directly:
index lists and thresholds must be bit-identical, for every key-range split (cluster
size), ragged row/key tiles, heavy ties, k = 1 and k = L."""

import numpy as np
import pytest
import torch

import oracle
from paper_2502_07590_b200 import ops

pytestmark = pytest.mark.gpu


def _operands(H, G, L, r, seed, ints=False, dev="cuda"):
    g = torch.Generator(device="cpu").manual_seed(seed)
    if ints:   # small integers: exact scores with massive ties
        q = torch.randint(-1, 2, (H, G, r), generator=g).float()
        k = torch.randint(-1, 2, (H, L, r), generator=g).float()
    else:
        q = torch.randn((H, G, r), generator=g)
        k = torch.randn((H, L, r), generator=g)
    return q.to(torch.bfloat16).to(dev), k.to(torch.bfloat16).to(dev)


def _compare(q, k, ks, split=0, check_oracle=False):
    for mode in ("fast", "multipass"):
        _compare_mode(q, k, ks, split, check_oracle, mode)


def _compare_mode(q, k, ks, split, check_oracle, mode):
    H, G, _ = q.shape
    L = k.shape[1]
    kc = torch.tensor(ks, dtype=torch.int32, device=q.device)
    kmax = max(ks)
    scores = ops.gemm_bf16(q, k, torch.float32)
    ref_idx, ref_thr = ops.topk_rows(scores.view(H * G, L), kc, G, kmax)
    idx, thr = ops.select_fused(q, k, kc, kmax, split=split, mode=mode)
    torch.cuda.synchronize()
    ri, rt, fi, ft = ref_idx.cpu().numpy(), ref_thr.cpu().numpy(), idx.cpu().numpy(), thr.cpu().numpy()
    for h in range(H):
        kh = ks[h]
        rows = slice(h * G, (h + 1) * G)
        np.testing.assert_array_equal(fi[rows, :kh], ri[rows, :kh],
                                      err_msg=f"head {h} k={kh} split={split} mode={mode}")
    assert np.all(ft == rt)
    if check_oracle:
        sc = scores.cpu().numpy()
        for h in range(H):
            oi, ot = oracle.topk_from_scores(sc[h], ks[h])
            np.testing.assert_array_equal(fi[h * G:(h + 1) * G, :ks[h]], oi)
            assert np.all(ft[h * G:(h + 1) * G] == ot.astype(np.float32))


@pytest.mark.parametrize("split", [1, 2, 3, 4, 0])
def test_fused_random_ragged(split):
    q, k = _operands(3, 200, 5000, 16, seed=split)
    _compare(q, k, [500, 1, 4999], split=split, check_oracle=(split == 2))


@pytest.mark.parametrize("split", [1, 3])
def test_fused_k_equals_L_and_tiny_L(split):
    q, k = _operands(2, 130, 390, 16, seed=7)
    _compare(q, k, [390, 389], split=split)
    q, k = _operands(1, 5, 1, 16, seed=8)
    _compare(q, k, [1], split=1)


@pytest.mark.parametrize("split", [1, 2, 4])
def test_fused_integer_ties(split):
    q, k = _operands(2, 256, 4096, 16, seed=11, ints=True)
    _compare(q, k, [410, 2048], split=split, check_oracle=True)


def test_fused_zero_scores_signed_zero():
    # all-zero query rows give +-0 scores everywhere: ties at 0 across the whole row
    q, k = _operands(1, 128, 3000, 16, seed=12)
    q[0, :64] = 0
    k[0, ::3] = -k[0, ::3]
    _compare(q, k, [300], split=2, check_oracle=True)


def test_fused_rank_not_16_and_strided_views():
    # r = 8 (zero-padded k-block) and the layer's strided [H, G, r] views of one projection
    H, G, L, r = 4, 260, 32760 // 8, 8
    g = torch.Generator(device="cpu").manual_seed(13)
    p = torch.randn((L, 2 * H * r), generator=g).to(torch.bfloat16).cuda()
    qp = p[:G, : H * r].view(G, H, r).permute(1, 0, 2)
    kl = p[:, H * r:].view(L, H, r).permute(1, 0, 2)
    _compare(qp, kl, [410, 1, 4000, 2000], split=0)


def test_fused_c2_shape():
    # c2: G = 260 proxy rows per head, L = 32760 keys, k = 3276 (90% sparsity)
    q, k = _operands(4, 260, 32760, 16, seed=14)
    _compare(q, k, [3276] * 4, split=0)


def test_fused_c5_row_length():
    # c5 row length (L = 524288), k = 52429, the extremes, and a tied row block
    q, k = _operands(3, 130, 524288, 16, seed=15)
    q[2, :40] = torch.round(q[2, :40] * 2) / 2
    _compare(q, k, [52429, 1, 524287], split=0)


def test_fast_mode_c2_needs_no_fallback():
    # c2's selection shape on random scores: the sampled band brackets every row's k-th
    # score, so the single-pass mode finishes every row tile itself
    q, k = _operands(24, 260, 32000, 16, seed=21)
    kc = torch.full((24,), 3200, dtype=torch.int32, device=q.device)
    ops.select_fused(q, k, kc, 3200, mode="fast")
    torch.cuda.synchronize()
    assert ops.select_fast_fallbacks(24, 260, 32000, 3200, 0, q.device) == 0


def test_resident_cluster_query():
    # the automatic split counts waves with resident clusters: one CTA per SM, fewer S-CTA
    # clusters than SMs / S where a GPC's SM count is not a multiple of S
    from paper_2502_07590_b200 import _lib

    lib = _lib.load()
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    n = [lib.dsv_select_fused_max_clusters(s) for s in range(1, 9)]
    assert n[0] == sms
    assert all(0 < n[s - 1] <= sms // s for s in range(1, 9))
    assert lib.dsv_select_fused_max_clusters(0) == 0 and lib.dsv_select_fused_max_clusters(9) == 0


@pytest.mark.parametrize("heads", [12, 6])
def test_auto_split_matches_forced(heads):
    # whatever split the occupancy rule picks, the selection is the same
    q, k = _operands(heads, 260, 32000, 16, seed=31)
    kc = torch.full((heads,), 3200, dtype=torch.int32, device=q.device)
    a = ops.select_fused(q, k, kc, 3200, split=0)
    b = ops.select_fused(q, k, kc, 3200, split=1)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
