"""Sampled sparsity profiler: oracle pinned to the reference's
golden vectors (tests/golden/profiler.npz from make_golden_profiler.py), the reference's own
known-answer cases, the host-side API, and the GPU path (dsv_critical_counts) against both."""

import numpy as np
import pytest
import torch

import oracle.profiler as OP
from conftest import GOLDEN
from paper_2502_07590_b200 import profiler as P


@pytest.fixture(scope="module")
def gp():
    return np.load(GOLDEN / "profiler.npz")


def _cases(gp, prefix):
    i = 0
    while f"{prefix}{i}_vals" in gp.files:
        yield i
        i += 1


# ---------------------------------------------------------------- oracle vs reference
def test_oracle_sample_queries_golden(gp):
    i = 0
    while f"sq{i}" in gp.files:
        s, f, seed = (int(x) for x in gp[f"sq{i}"])
        np.testing.assert_array_equal(OP.sample_queries(s, f, seed), gp[f"sq{i}_rows"])
        np.testing.assert_array_equal(P.sample_queries(s, P.SampleConfig(factor=f), seed=seed),
                                      gp[f"sq{i}_rows"])
        i += 1


@pytest.mark.parametrize("prefix", ["mb", "mi"])
def test_oracle_measure_block_sparsity_golden(gp, prefix):
    for i in _cases(gp, prefix):
        theta, f, seed = gp[f"{prefix}{i}_meta"]
        vals = OP.measure_block_sparsity(list(gp[f"{prefix}{i}_q"]), list(gp[f"{prefix}{i}_k"]),
                                         theta, int(f), int(seed))
        np.testing.assert_allclose(vals, gp[f"{prefix}{i}_vals"], rtol=0, atol=1e-12)


def test_oracle_critical_sizes_golden(gp):
    for i in _cases(gp, "mi"):
        theta, f, seed = gp[f"mi{i}_meta"]
        q, k = gp[f"mi{i}_q"][0], gp[f"mi{i}_k"][0]
        rows = OP.sample_queries(q.shape[0], int(f), int(seed))
        p = OP.softmax_rows(q[rows] @ k.T / np.sqrt(q.shape[1]))
        np.testing.assert_array_equal(OP.critical_counts(p, theta), gp[f"mi{i}_sizes0"])


def test_oracle_reference_known_answers():
    # tests/test_profiler.py:62-80 of the reference
    s = 100
    rng = np.random.default_rng(0)
    q = np.zeros((s, 4))
    q[:, 0] = 50.0
    k = rng.standard_normal((s, 4)) * 0.01
    k[7, 0] = 10.0
    assert OP.measure_block_sparsity([q], [k], 0.9, 1, 0)[0] == pytest.approx(0.99)
    z = np.zeros((s, 3))
    assert OP.measure_block_sparsity([z], [z], 0.9, 1, 0)[0] == pytest.approx(1 - np.ceil(0.9 * s) / s)


# ---------------------------------------------------------------- host API
def test_sample_config_validation():
    with pytest.raises(ValueError):
        P.SampleConfig(factor=0)
    with pytest.raises(ValueError):
        P.SampleConfig(stage1_period=0)
    with pytest.raises(ValueError):
        P.sample_queries(10, P.SampleConfig(factor=16))


def test_ema_and_profile():
    assert P.ema_update(0.8, 0.9, 0.1) == pytest.approx(0.81)
    assert P.ema_update(0.3, 0.7, 1.0) == pytest.approx(0.7)
    with pytest.raises(ValueError):
        P.ema_update(0.5, 0.5, 0.0)
    prof = P.SparsityProfile(alpha=0.5)
    prof.update_block(0, [0.9, 0.8], 1)
    prof.update_block(0, [0.7, 0.6], 2)
    np.testing.assert_allclose(prof.head_emas(0), [0.8, 0.7])
    again = P.SparsityProfile.from_snapshot(prof.snapshot())
    assert again.snapshot() == prof.snapshot()
    assert prof.blocks() == [0] and prof.block_mean(0) == pytest.approx(0.75)


# ---------------------------------------------------------------- GPU path
@pytest.mark.gpu
def test_gpu_profiler_integer_inputs_exact(cuda, gp):
    for i in _cases(gp, "mi"):
        theta, f, seed = gp[f"mi{i}_meta"]
        qs = [torch.from_numpy(x.astype(np.float32)).to(cuda) for x in gp[f"mi{i}_q"]]
        ks = [torch.from_numpy(x.astype(np.float32)).to(cuda) for x in gp[f"mi{i}_k"]]
        vals = P.measure_block_sparsity(qs, ks, theta, P.SampleConfig(factor=int(f)), seed=int(seed))
        # the per-row counts are exact (next test); only the mean's summation order differs
        np.testing.assert_allclose(vals, gp[f"mi{i}_vals"], rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_gpu_critical_counts_match_oracle_rows(cuda, gp):
    from paper_2502_07590_b200 import ops

    for i in _cases(gp, "mi"):
        theta, f, seed = gp[f"mi{i}_meta"]
        q, k = gp[f"mi{i}_q"][0], gp[f"mi{i}_k"][0]
        rows = OP.sample_queries(q.shape[0], int(f), int(seed))
        x = torch.from_numpy((q[rows] @ k.T).astype(np.float32)).to(cuda)
        n = ops.critical_counts(x, float(np.sqrt(q.shape[1])), float(theta)).cpu().numpy()
        np.testing.assert_array_equal(n, gp[f"mi{i}_sizes0"])


@pytest.mark.gpu
def test_gpu_profiler_random_inputs(cuda, gp):
    # fp32 logits on the GPU vs fp64 in the reference: a row's prefix length can move
    # by one at a mass boundary; the per-head sparsity stays within a few 1/S
    for i in _cases(gp, "mb"):
        theta, f, seed = gp[f"mb{i}_meta"]
        qs = [torch.from_numpy(x.astype(np.float32)).to(cuda) for x in gp[f"mb{i}_q"]]
        ks = [torch.from_numpy(x.astype(np.float32)).to(cuda) for x in gp[f"mb{i}_k"]]
        vals = P.measure_block_sparsity(qs, ks, theta, P.SampleConfig(factor=int(f), seed=int(seed)))
        s = gp[f"mb{i}_q"].shape[1]
        np.testing.assert_allclose(vals, gp[f"mb{i}_vals"], rtol=0, atol=2.0 / s)


@pytest.mark.gpu
def test_gpu_profiler_known_answers_and_bf16(cuda):
    s = 100
    rng = np.random.default_rng(0)
    q = np.zeros((s, 4), np.float32)
    q[:, 0] = 50.0
    k = (rng.standard_normal((s, 4)) * 0.01).astype(np.float32)
    k[7, 0] = 10.0
    cfg = P.SampleConfig(factor=1)
    assert P.measure_block_sparsity([q], [k], 0.9, cfg)[0] == pytest.approx(0.99)
    z = np.zeros((s, 3), np.float32)
    assert P.measure_block_sparsity([z], [z], 0.9, cfg)[0] == pytest.approx(1 - np.ceil(0.9 * s) / s)
    # bf16 operands (tcgen05 scores): vs the oracle on the same bf16-rounded values
    S, d = 4096, 64
    qb = torch.randn((S, d), device=cuda).to(torch.bfloat16)
    kb = torch.randn((S, d), device=cuda).to(torch.bfloat16)
    got = P.measure_block_sparsity([qb], [kb], 0.9, P.SampleConfig(factor=16))[0]
    ref = OP.measure_block_sparsity([qb.float().cpu().numpy()], [kb.float().cpu().numpy()], 0.9, 16, 0)[0]
    assert abs(got - ref) <= 2.0 / S
