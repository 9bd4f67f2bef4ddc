"""Full/sparse dispatcher: the model time source and the decision
rule reproduce the reference exactly (tests/golden/dispatcher.npz from
make_golden_dispatcher.py); the GPU time source calibrates on the device kernels."""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2502_07590_b200 import dispatcher as DP

FIELDS = ("length", "sparsity", "full_time", "sparse_time", "estimation_time", "index_bytes",
          "full_flops", "sparse_flops", "estimation_flops", "selection_flops")
REASONS = {"enabled": 0, "sparsity below threshold": 1, "memory exceeded": 2}


@pytest.fixture(scope="module")
def gd():
    return np.load(GOLDEN / "dispatcher.npz")


def test_model_table_and_decisions_match_reference(gd, tmp_path):
    t = DP.calibrate([256, 1000, 4096], [0.0, 0.5, 0.9, 0.93], d_k=64, d_lr=16, time_source="model")
    got = np.array([[float(getattr(t.entries[k], f)) for f in FIELDS] for k in sorted(t.entries)])
    np.testing.assert_array_equal(got, gd["table"])
    np.testing.assert_array_equal([t.crossover(l) for l in t.lengths()], gd["crossover"])
    for s, length, mem, en, reason, k, bucket, fb in gd["decide"]:
        d = DP.decide(float(s), int(length), int(mem), t)
        assert (int(d.enabled), REASONS[d.reason], d.k, d.length_bucket, int(d.bucket_fallback)) == \
            (int(en), int(reason), int(k), int(bucket), int(fb))
    assert [DP.serialized_index_bytes(64, 7, 4), DP.serialized_index_bytes(10, 3, 8)] == list(gd["ser_bytes"])
    p = tmp_path / "t.csv"
    t.to_csv(p)
    back = DP.CostProfileTable.from_csv(p)
    assert back.entries == t.entries


def test_buckets_and_errors():
    assert DP.length_bucket(513) == 1024 and DP.sparsity_bucket(0.93) == pytest.approx(0.9)
    with pytest.raises(ValueError):
        DP.calibrate([], [0.5])
    with pytest.raises(ValueError):
        DP.calibrate([256], [0.5], time_source="nope")
    with pytest.raises(ValueError):
        DP.decide(1.0, 100, 1, DP.calibrate([256], [0.5], time_source="model"))


@pytest.mark.gpu
def test_gpu_calibration(cuda):
    t = DP.calibrate([1024, 16384], [0.0, 0.5, 0.9, 0.95], reps=3, d_k=128, time_source="gpu")
    for e in t.entries.values():
        assert e.full_time > 0 and e.sparse_time > 0 and e.estimation_time > 0
    # sparse attention at 95% sparsity beats the dense path at 16k tokens on the device
    e = t.entries[(16384, 0.95)]
    assert e.sparse_time < e.full_time
    assert t.crossover(16384) is not None and t.crossover(16384) <= 0.95
    d = DP.decide(0.95, 16384, 10**12, t)
    assert d.enabled and d.reason == "enabled"
