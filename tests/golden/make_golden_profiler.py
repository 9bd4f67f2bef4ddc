"""Golden vectors for the sampled sparsity profiler, produced by running the REFERENCE
(pkg/src/dynsparse/profiler.py, attention.py) in the build container:
    python tests/golden/make_golden_profiler.py
Writes tests/golden/profiler.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    from dynsparse import attention as A
    from dynsparse import profiler as P

    rng = np.random.default_rng(11)
    g = {}
    cases = [(100, 16, 0), (1024, 16, 3), (4096, 16, 0), (77, 1, 5), (500, 7, 9)]
    for i, (s, f, seed) in enumerate(cases):
        g[f"sq{i}"] = np.array([s, f, seed])
        g[f"sq{i}_rows"] = P.sample_queries(s, P.SampleConfig(factor=f), seed=seed)
    # random heads (fp32-representable inputs), several theta / factors
    for i, (s, d, theta, f, scale) in enumerate([(256, 16, 0.9, 1, 1.0), (512, 8, 0.5, 4, 2.0),
                                                 (1024, 32, 0.95, 16, 1.5), (300, 16, 0.99, 2, 3.0)]):
        qs = [(scale * rng.standard_normal((s, d))).astype(np.float32).astype(np.float64) for _ in range(3)]
        ks = [(scale * rng.standard_normal((s, d))).astype(np.float32).astype(np.float64) for _ in range(3)]
        vals = P.measure_block_sparsity(qs, ks, theta, P.SampleConfig(factor=f, seed=i))
        g[f"mb{i}_q"], g[f"mb{i}_k"] = np.stack(qs), np.stack(ks)
        g[f"mb{i}_meta"] = np.array([theta, f, i], dtype=np.float64)
        g[f"mb{i}_vals"] = vals
    # integer-valued inputs: exact logits in fp32 and fp64 (heavy ties)
    for i, (s, d, theta, f) in enumerate([(256, 4, 0.9, 1), (640, 8, 0.7, 5)]):
        qs = [rng.integers(-2, 3, size=(s, d)).astype(np.float64) for _ in range(2)]
        ks = [rng.integers(-2, 3, size=(s, d)).astype(np.float64) for _ in range(2)]
        vals = P.measure_block_sparsity(qs, ks, theta, P.SampleConfig(factor=f, seed=7))
        g[f"mi{i}_q"], g[f"mi{i}_k"] = np.stack(qs), np.stack(ks)
        g[f"mi{i}_meta"] = np.array([theta, f, 7], dtype=np.float64)
        g[f"mi{i}_vals"] = vals
        # the per-row oracle set sizes of head 0 (sampled rows)
        rows = P.sample_queries(s, P.SampleConfig(factor=f, seed=7))
        sc = A.attention_scores(qs[0][rows], ks[0])
        g[f"mi{i}_sizes0"] = A.critical_kv_oracle(sc, theta).sizes()
    np.savez_compressed(OUT / "profiler.npz", **g)
    print("wrote", OUT / "profiler.npz")


if __name__ == "__main__":
    main()
