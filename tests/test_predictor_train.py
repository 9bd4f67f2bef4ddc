"""Predictor training step: oracle pinned to the reference
(tests/golden/predictor.npz from make_golden_predictor.py), then the device path
(dsv_pred_pass + fp64 library GEMMs) against the same vectors and the reference's own
known-answer cases (predictor tests: zero params, non-finite skip, teacher convergence)."""

import numpy as np
import pytest
import torch

import oracle.predictor as OPR
from conftest import GOLDEN


@pytest.fixture(scope="module")
def gpr():
    return np.load(GOLDEN / "predictor.npz")


def _case(g, i):
    rows = g[f"c{i}_rows"]
    return (g[f"c{i}_wq"], g[f"c{i}_wk"], g[f"c{i}_x"], g[f"c{i}_t"], None if rows[0] < 0 else rows)


def _n(g):
    return sum(1 for k in g.files if k.endswith("_loss"))


def test_oracle_matches_reference(gpr):
    for i in range(_n(gpr)):
        wq, wk, x, t, rows = _case(gpr, i)
        cl, nl, tot, gq, gk = OPR.loss_and_grads(wq, wk, x, t, rows)
        np.testing.assert_array_equal([cl, nl, tot], gpr[f"c{i}_loss"])
        np.testing.assert_array_equal(gq, gpr[f"c{i}_gq"])
        np.testing.assert_array_equal(gk, gpr[f"c{i}_gk"])
        wq10, wk10, hist = OPR.train(wq, wk, x, t, 10, lr=3e-3, rows=rows)
        np.testing.assert_array_equal(hist, gpr[f"c{i}_hist"])
        np.testing.assert_array_equal(wq10, gpr[f"c{i}_wq10"])


def test_predictor_loss_host(gpr):
    from paper_2502_07590_b200.predictor import predictor_loss

    rng = np.random.default_rng(0)
    a, t = rng.standard_normal((6, 8)), rng.standard_normal((6, 8))
    t[2] = 0.0
    rep = predictor_loss(a, t)
    cl, _ = OPR.cos_terms(a, t)
    nl, _ = OPR.norm_terms(a, t)
    assert rep.cos_loss == pytest.approx(cl, rel=1e-12) and rep.norm_loss == pytest.approx(nl, rel=1e-12)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.gpu
def test_gpu_loss_and_grads_match_reference(cuda, gpr):
    from paper_2502_07590_b200.predictor import PredictorParams, loss_and_grads

    for i in range(_n(gpr)):
        wq, wk, x, t, rows = _case(gpr, i)
        p = PredictorParams(w_q=wq.copy(), w_k=wk.copy())
        rep, gq, gk = loss_and_grads(p, x, t, rows=rows)
        np.testing.assert_allclose([rep.cos_loss, rep.norm_loss, rep.total], gpr[f"c{i}_loss"], rtol=1e-10)
        assert _rel(gq, gpr[f"c{i}_gq"]) < 1e-9 and _rel(gk, gpr[f"c{i}_gk"]) < 1e-9
        # fp32 target on the device: vs the oracle on the same fp32-rounded target
        t32 = torch.from_numpy(t.astype(np.float32)).to(cuda)
        rep32, gq32, gk32 = loss_and_grads(p, x, t32, rows=rows)
        cl, nl, tot, oq, ok = OPR.loss_and_grads(wq, wk, x, t.astype(np.float32).astype(np.float64), rows)
        assert rep32.total == pytest.approx(tot, rel=1e-10)
        assert _rel(gq32, oq) < 1e-9 and _rel(gk32, ok) < 1e-9


@pytest.mark.gpu
def test_gpu_train_steps_match_reference(cuda, gpr):
    from paper_2502_07590_b200.predictor import PredictorParams, train_step

    for i in range(_n(gpr)):
        wq, wk, x, t, rows = _case(gpr, i)
        p = PredictorParams(w_q=wq.copy(), w_k=wk.copy(), lr=3e-3)
        hist = [train_step(p, x, t, rows=rows).total for _ in range(10)]
        np.testing.assert_allclose(hist, gpr[f"c{i}_hist"], rtol=1e-9)
        assert _rel(p.w_q, gpr[f"c{i}_wq10"]) < 1e-9 and _rel(p.w_k, gpr[f"c{i}_wk10"]) < 1e-9


@pytest.mark.gpu
def test_gpu_reference_known_answers(cuda):
    from paper_2502_07590_b200.predictor import PredictorParams, loss_and_grads, train_step

    rng = np.random.default_rng(0)
    # zero params and zero target: zero gradients, no update (reference test_zero_params_zero_target)
    p = PredictorParams(w_q=np.zeros((4, 2)), w_k=np.zeros((4, 2)))
    x = rng.standard_normal((6, 4))
    _, gq, gk = loss_and_grads(p, x, np.zeros((6, 6)))
    assert not gq.any() and not gk.any()
    train_step(p, x, np.zeros((6, 6)))
    assert not p.w_q.any() and not p.w_k.any()
    # non-finite forward product: the step is skipped (test_nonfinite_gradient_skips_step)
    p = PredictorParams.initialize(4, 2, seed=0)
    p.w_q *= 1e308
    before = p.w_q.copy()
    with np.errstate(all="ignore"):
        rep = train_step(p, rng.standard_normal((4, 4)), rng.standard_normal((4, 4)))
    assert rep.step_skipped and np.array_equal(p.w_q, before)


@pytest.mark.gpu
def test_gpu_teacher_convergence(cuda):
    # reference TestTrainingAndEstimation.test_teacher_convergence_and_recall (training half)
    from paper_2502_07590_b200.predictor import PredictorParams, train_step

    rng = np.random.default_rng(42)
    s, d, d_lr = 256, 32, 16
    x = rng.standard_normal((s, d))
    a_t = rng.standard_normal((d, 4)) / np.sqrt(d)
    b_t = rng.standard_normal((d, 4)) / np.sqrt(d)
    target = (x @ a_t) @ (x @ b_t).T
    p = PredictorParams.initialize(d, d_lr, seed=7, lr=1e-3)
    tgt = torch.from_numpy(target).to(cuda)
    rep = None
    for _ in range(2000):
        rep = train_step(p, x, tgt)
        if rep.total < 0.005:
            break
    assert rep.total < 0.01
