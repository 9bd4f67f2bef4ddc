"""Pin the CPU oracle to golden vectors produced by the reference itself
(tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

import oracle
from conftest import GOLDEN


@pytest.fixture(scope="module")
def sel():
    return np.load(GOLDEN / "selection.npz")


def test_k_from_sparsity_table(sel):
    for (s, n), k in zip(sel["kfs_args"], sel["kfs_k"]):
        assert oracle.k_from_sparsity(s, int(n)) == k


def test_topk_lowrank_random(sel):
    idx, thr = oracle.topk_lowrank(sel["rand_q"], sel["rand_k"], 9)
    np.testing.assert_array_equal(idx, sel["rand_idx"])
    np.testing.assert_array_equal(idx, sel["rand_idx_twopass"])
    np.testing.assert_allclose(thr, sel["rand_thr"], rtol=1e-12)


def test_topk_lowrank_heavy_ties(sel):
    idx, thr = oracle.topk_lowrank(sel["ties_q"], sel["ties_k"], 30)
    np.testing.assert_array_equal(idx, sel["ties_idx"])
    np.testing.assert_array_equal(idx, sel["ties_idx_twopass"])
    np.testing.assert_array_equal(thr, sel["ties_thr"])


@pytest.mark.parametrize("k", [1, 7, 120, 499, 500])
def test_topk_given_scores_signed_zero_ties(sel, k):
    idx, thr = oracle.topk_from_scores(sel["given_scores"], k)
    np.testing.assert_array_equal(idx, sel[f"given_idx_{k}"])
    np.testing.assert_array_equal(thr, sel[f"given_thr_{k}"])   # == treats -0.0 == +0.0


def test_topk_rejects_bad_k():
    with pytest.raises(ValueError):
        oracle.topk_from_scores(np.zeros((2, 3)), 4)
    with pytest.raises(ValueError):
        oracle.topk_from_scores(np.zeros((2, 3)), 0)


def test_attention_golden():
    g = np.load(GOLDEN / "attention.npz")
    np.testing.assert_allclose(oracle.full_attention(g["q"], g["k"], g["v"]), g["full"], atol=1e-12)
    uni = list(g["uni_idx"])
    out, _ = oracle.rows_attention_fwd(g["q"], g["k"], g["v"], uni)
    np.testing.assert_allclose(out, g["uni_out"], atol=1e-12)
    ptr, cols = g["rag_ptr"], g["rag_cols"]
    rag = [cols[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
    out, _ = oracle.rows_attention_fwd(g["q"], g["k"], g["v"], rag)
    np.testing.assert_allclose(out, g["rag_out"], atol=1e-12)


def test_grouping_golden():
    g = np.load(GOLDEN / "grouping.npz")
    i = 0
    while f"c{i}_grid" in g:
        members, proxies = oracle.build_groups(g[f"c{i}_grid"], g[f"c{i}_dims"])
        np.testing.assert_array_equal(proxies, g[f"c{i}_proxies"])
        np.testing.assert_array_equal([m.size for m in members], g[f"c{i}_sizes"])
        np.testing.assert_array_equal(np.concatenate(members), g[f"c{i}_members"])
        i += 1
    assert i >= 6
    members, _ = oracle.build_groups((2, 4, 4), (2, 2, 2))
    ptr, cols = g["ga_ptr"], g["ga_cols"]
    sets = [cols[ptr[j]:ptr[j + 1]] for j in range(len(ptr) - 1)]
    out, _ = oracle.grouped_attention_fwd(g["ga_q"], g["ga_k"], g["ga_v"], members, sets)
    np.testing.assert_allclose(out, g["ga_out"], atol=1e-12)


def test_backward_matches_trainer_autograd():
    g = np.load(GOLDEN / "backward.npz")
    B, S, H, dk = (int(x) for x in g["shape"])
    x = g["x"].reshape(B, S, 3, H, dk)
    dx = g["dx"].reshape(B, S, 3, H, dk)
    dout = g["dout"].reshape(B, S, H, dk)
    out_ref = g["out"].reshape(B, S, H, dk)
    for b in range(B):
        lists = [g["idx"][b, s] for s in range(S)]
        for h in range(H):
            q, k, v = x[b, :, 0, h], x[b, :, 1, h], x[b, :, 2, h]
            out, _ = oracle.rows_attention_fwd(q, k, v, lists)
            np.testing.assert_allclose(out, out_ref[b, :, h], atol=1e-12)
            dq, dk_, dv = oracle.rows_attention_bwd(q, k, v, lists, dout[b, :, h])
            np.testing.assert_allclose(dq, dx[b, :, 0, h], atol=1e-10)
            np.testing.assert_allclose(dk_, dx[b, :, 1, h], atol=1e-10)
            np.testing.assert_allclose(dv, dx[b, :, 2, h], atol=1e-10)
