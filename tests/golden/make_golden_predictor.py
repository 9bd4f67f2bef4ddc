"""Golden vectors for the predictor training step, produced by running the REFERENCE
(pkg/src/dynsparse/predictor.py) in the build container:
    python tests/golden/make_golden_predictor.py
Writes tests/golden/predictor.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    from dynsparse import predictor as PR

    rng = np.random.default_rng(5)
    g = {}
    cases = [(64, 16, 4, None), (200, 32, 16, 10), (96, 12, 8, 3), (300, 24, 16, 16)]
    for i, (s, d, r, factor) in enumerate(cases):
        x = rng.standard_normal((s, d))
        rows = None if factor is None else np.sort(rng.choice(s, size=-(-s // factor), replace=False))
        nr = s if rows is None else rows.size
        target = rng.standard_normal((nr, s)) * 3.0
        if i == 2:
            target[1] = 0.0                       # a zero target row (skipped, still counted)
        p = PR.PredictorParams.initialize(d, r, seed=i)
        rep, gq, gk = PR.loss_and_grads(p, x, target, rows=rows)
        g[f"c{i}_x"], g[f"c{i}_t"], g[f"c{i}_wq"], g[f"c{i}_wk"] = x, target, p.w_q, p.w_k
        g[f"c{i}_rows"] = np.array([-1]) if rows is None else rows
        g[f"c{i}_loss"] = np.array([rep.cos_loss, rep.norm_loss, rep.total])
        g[f"c{i}_gq"], g[f"c{i}_gk"] = gq, gk
        # ten Adam steps
        p2 = PR.PredictorParams.initialize(d, r, seed=i, lr=3e-3)
        hist = [PR.train_step(p2, x, target, rows=rows).total for _ in range(10)]
        g[f"c{i}_hist"], g[f"c{i}_wq10"], g[f"c{i}_wk10"] = np.array(hist), p2.w_q, p2.w_k
    np.savez_compressed(OUT / "predictor.npz", **g)
    print("wrote", OUT / "predictor.npz")


if __name__ == "__main__":
    main()
