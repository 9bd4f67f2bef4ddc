"""The reference-precision (fp64) path of the reference-named API against the oracle and the
reference's goldens: host fp64 callers get the reference's own tolerances (1e-12 .. 1e-9).

  * dsv_topk_f64: bit-exact indices, thresholds == the oracle's on the same fp64 scores
    (random, integer ties, +-0.0, per-row k, rows past the CTA size);
  * dsv_gemm_f64 / project: exact for identity / zero / integer operands, 1e-12 otherwise;
  * dsv_rows_*_f64 (sparse / full attention, d_v != d_k): <= 1e-12 vs the fp64 oracle;
  * critical_kv_oracle / analyze_distribution / attention_scores / prediction_accuracy /
    select_group_critical: the reference's rule restated in oracle/profiler.py.
"""

import numpy as np
import pytest
import torch

import oracle
from oracle.profiler import critical_counts, softmax_rows
from paper_2502_07590_b200 import ops
from paper_2502_07590_b200.attention import (CriticalIndexSet, analyze_distribution,
                                             attention_scores, critical_kv_oracle, full_attention,
                                             sparse_attention)
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.grouping import build_groups, select_group_critical
from paper_2502_07590_b200.predictor import (PredictorParams, estimate_critical,
                                             prediction_accuracy, project)
from paper_2502_07590_b200.selection import AllocationMeter, streaming_topk

pytestmark = pytest.mark.gpu


def _topk_dev(scores, ks, rows_per_k):
    s = torch.from_numpy(np.ascontiguousarray(scores, dtype=np.float64)).cuda()
    kp = torch.tensor(ks, dtype=torch.int32, device="cuda")
    idx, thr = ops.topk_f64(s, kp, rows_per_k, max(ks))
    return idx.cpu().numpy(), thr.cpu().numpy()


@pytest.mark.parametrize("L", [1, 5, 255, 256, 257, 1000, 4096, 70000])
def test_topk_f64_random_matches_oracle(cuda, L):
    rng = np.random.default_rng(L)
    sc = rng.standard_normal((12, L))
    ks = [int(x) for x in rng.integers(1, L + 1, size=3)]
    idx, thr = _topk_dev(sc, ks, 4)
    per = np.repeat(ks, 4)
    ri, rt = oracle.topk_from_scores(sc, per)
    for r in range(12):
        np.testing.assert_array_equal(idx[r, : per[r]], ri[r, : per[r]])
    np.testing.assert_array_equal(thr, rt)


def test_topk_f64_ties_and_signed_zero(cuda):
    rng = np.random.default_rng(3)
    sc = rng.integers(-3, 4, size=(20, 3000)).astype(np.float64)
    sc[0] = 0.0
    sc[1, ::2] = -0.0
    sc[2] = 1.0
    for k in (1, 7, 1500, 2999, 3000):
        idx, thr = _topk_dev(sc, [k], 20)
        ri, rt = oracle.topk_from_scores(sc, k)
        np.testing.assert_array_equal(idx[:, :k], ri)
        assert np.all(thr == rt)


def test_project_exact_and_precise(cuda):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((37, 19))
    np.testing.assert_array_equal(project(x, np.eye(19)), x)
    np.testing.assert_array_equal(project(x, np.zeros((19, 5))), np.zeros((37, 5)))
    w = rng.standard_normal((19, 7))
    np.testing.assert_allclose(project(x, w), x @ w, atol=1e-12)
    assert project(x.astype(np.float32), w.astype(np.float32)).dtype == np.float32


def test_streaming_topk_fp64_thresholds(cuda):
    rng = np.random.default_rng(99)
    for _ in range(10):
        sq, sk, d = int(rng.integers(1, 64)), int(rng.integers(2, 96)), int(rng.integers(1, 8))
        k = int(rng.integers(1, min(sk, 24) + 1))
        q, kk = rng.standard_normal((sq, d)), rng.standard_normal((sk, d))
        got = streaming_topk(q, kk, k)
        ri, rt = oracle.topk_lowrank(q, kk, k)
        np.testing.assert_array_equal(got.indices, ri)
        np.testing.assert_allclose(got.thresholds, rt, rtol=1e-12)


def test_allocation_meter_reference_bound(cuda):
    rng = np.random.default_rng(1)
    s, k = 1024, 32
    meter = AllocationMeter()
    streaming_topk(rng.standard_normal((s, 8)), rng.standard_normal((s, 8)), k, meter=meter)
    assert meter.peak <= 8 * s * k
    assert meter.current == 0


@pytest.mark.parametrize("dk,dv", [(8, 8), (64, 64), (5, 11), (128, 40)])
def test_attention_f64_matches_oracle(cuda, dk, dv):
    rng = np.random.default_rng(dk * 7 + dv)
    S = 50
    q, k = rng.standard_normal((S, dk)), rng.standard_normal((S, dk))
    v = rng.standard_normal((S, dv))
    lists = [np.sort(rng.choice(S, size=int(rng.integers(1, S + 1)), replace=False)) for _ in range(S)]
    got = sparse_attention(q, k, v, CriticalIndexSet(lists))
    ref, _ = oracle.rows_attention_fwd(q, k, v, lists)
    np.testing.assert_allclose(got, ref, atol=1e-12)
    full = full_attention(q, k, v)
    np.testing.assert_allclose(full, softmax_rows(q @ k.T / np.sqrt(dk)) @ v, atol=1e-12)
    assert got.dtype == np.float64


def test_rows_bwd_f64_matches_oracle(cuda):
    rng = np.random.default_rng(5)
    S, D = 40, 16
    q, k, v, do = (rng.standard_normal((S, D)) for _ in range(4))
    lists = [np.sort(rng.choice(S, size=int(rng.integers(1, S + 1)), replace=False)) for _ in range(S)]
    ptr = torch.from_numpy(np.concatenate([[0], np.cumsum([x.size for x in lists])])).cuda()
    cols = torch.from_numpy(np.concatenate(lists).astype(np.int32)).cuda()
    t = [torch.from_numpy(x)[None].cuda() for x in (q, k, v, do)]
    out, lse = ops.rows_fwd_f64(t[0], t[1], t[2], ptr, cols, 1 / np.sqrt(D))
    dq, dk, dv = ops.rows_bwd_f64(t[0], t[1], t[2], out, lse, t[3], ptr, cols, 1 / np.sqrt(D))
    rdq, rdk, rdv = oracle.rows_attention_bwd(q, k, v, lists, do)
    for got, ref in ((dq, rdq), (dk, rdk), (dv, rdv)):
        np.testing.assert_allclose(got[0].cpu().numpy(), ref, atol=1e-12)


@pytest.mark.parametrize("S,theta", [(64, 0.9), (300, 0.5), (1, 0.9), (2049, 0.95), (20000, 0.8)])
def test_critical_kv_oracle_matches_reference_rule(cuda, S, theta):
    rng = np.random.default_rng(S)
    R = 6
    q, k = rng.standard_normal((R, 16)), rng.standard_normal((S, 16))
    scores = softmax_rows(q @ k.T / 4.0)
    scores[0, :] = 1.0 / S                       # all tied: lowest indices first
    sets = critical_kv_oracle(scores, theta)
    counts = critical_counts(scores, theta)
    cols = np.arange(S)
    for r in range(R):
        order = np.lexsort((cols, -scores[r]))
        np.testing.assert_array_equal(sets.indices[r], np.sort(order[: counts[r]]))


def test_attention_scores_and_distribution(cuda):
    rng = np.random.default_rng(2)
    grid = TokenGrid(2, 4, 8)
    S = grid.size
    q, k = rng.standard_normal((S, 8)), rng.standard_normal((S, 8))
    sc = attention_scores(q, k)
    np.testing.assert_allclose(sc, softmax_rows(q @ k.T / np.sqrt(8)), atol=1e-14)
    np.testing.assert_allclose(sc.sum(axis=1), 1.0, atol=1e-12)
    rep = analyze_distribution(sc, grid, theta=0.9, top_fraction=0.1)
    top_n = int(np.ceil(0.1 * S))
    np.testing.assert_allclose(rep["top_mass_fraction_mean"],
                               np.mean(np.sort(sc, axis=1)[:, ::-1][:, :top_n].sum(axis=1)), rtol=1e-12)
    edges = np.asarray(rep["histogram"]["edges"])
    np.testing.assert_array_equal(rep["histogram"]["counts"], np.histogram(sc, bins=edges)[0])
    assert 0 < rep["critical_kv"]["mean_distance"]


def test_prediction_accuracy_and_group_critical(cuda):
    rng = np.random.default_rng(4)
    grid = TokenGrid(2, 4, 8)
    S = grid.size
    x = rng.standard_normal((S, 32))
    params = PredictorParams.initialize(32, 4, seed=1)
    est = estimate_critical(params, x, k=6)
    q, k = rng.standard_normal((S, 16)), rng.standard_normal((S, 16))
    sc = softmax_rows(q @ k.T / 4.0)
    ora = critical_kv_oracle(sc, 0.9)
    rec, cov = prediction_accuracy(est, ora, sc)
    recs = [np.intersect1d(e, o).size / o.size for e, o in zip(est.indices, ora.indices)]
    covs = [sc[i, e].sum() / sc[i, o].sum() for i, (e, o) in enumerate(zip(est.indices, ora.indices))]
    assert rec == pytest.approx(np.mean(recs), rel=1e-12)
    assert cov == pytest.approx(np.mean(covs), rel=1e-12)
    plan = build_groups(grid, (2, 2, 2))
    sets = select_group_critical(q, k, plan, 0.9)
    psc = softmax_rows(q[plan.proxies] @ k.T / 4.0)
    counts = critical_counts(psc, 0.9)
    for g, sel in enumerate(sets):
        order = np.lexsort((np.arange(S), -psc[g]))
        np.testing.assert_array_equal(sel, np.sort(order[: counts[g]]))
