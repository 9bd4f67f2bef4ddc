"""Golden vectors for the dispatcher (model time source and decisions), produced by running
the REFERENCE (pkg/src/dynsparse/dispatcher.py) in the build container:
    python tests/golden/make_golden_dispatcher.py
Writes tests/golden/dispatcher.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
FIELDS = ("length", "sparsity", "full_time", "sparse_time", "estimation_time", "index_bytes",
          "full_flops", "sparse_flops", "estimation_flops", "selection_flops")


def main():
    sys.path.insert(0, str(REF))
    from dynsparse import dispatcher as D

    t = D.calibrate([256, 1000, 4096], [0.0, 0.5, 0.9, 0.93], d_k=64, d_lr=16, time_source="model")
    keys = sorted(t.entries)
    g = {"table": np.array([[float(getattr(t.entries[k], f)) for f in FIELDS] for k in keys])}
    cases = [(0.95, 4096, 10**9), (0.5, 4096, 10**9), (0.9, 3000, 10**9), (0.92, 700, 10**9),
             (0.99, 4096, 1000), (0.0, 256, 10**9), (0.9, 100000, 10**12)]
    dec = []
    for s, length, mem in cases:
        d = D.decide(s, length, mem, t)
        dec.append([s, length, mem, int(d.enabled), {"enabled": 0, "sparsity below threshold": 1,
                                                    "memory exceeded": 2}[d.reason], d.k, d.length_bucket,
                    int(d.bucket_fallback)])
    g["decide"] = np.array(dec, dtype=np.float64)
    g["crossover"] = np.array([t.crossover(l) if t.crossover(l) is not None else -1.0 for l in t.lengths()])
    g["ser_bytes"] = np.array([D.serialized_index_bytes(64, 7, 4), D.serialized_index_bytes(10, 3, 8)])
    np.savez_compressed(OUT / "dispatcher.npz", **g)
    print("wrote", OUT / "dispatcher.npz")


if __name__ == "__main__":
    main()
