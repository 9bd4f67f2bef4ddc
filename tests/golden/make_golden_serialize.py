"""Golden vectors for the index-set wire formats, produced by running the REFERENCE
(pkg/src/dynsparse/serialize.py) in the build container:
    python tests/golden/make_golden_serialize.py
Writes tests/golden/serialize.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    from dynsparse import serialize as SE

    rng = np.random.default_rng(3)
    g = {}
    sets = []
    # ragged sorted rows over a range that needs 1-4 byte varints (first values and gaps)
    for i in range(40):
        n = int(rng.integers(0, 300))
        hi = [200, 20000, 3000000, 200000000][i % 4]
        sets.append(np.sort(rng.choice(hi, size=min(n, hi), replace=False)))
    ptr = np.cumsum([0] + [len(r) for r in sets])
    g["ptr"], g["cols"] = ptr, np.concatenate(sets)
    g["varint"] = np.frombuffer(SE.encode_index_sets(sets), dtype=np.uint8)
    g["raw4"] = np.frombuffer(SE.raw_index_payload(sets, 4), dtype=np.uint8)
    g["raw8"] = np.frombuffer(SE.raw_index_payload(sets, 8), dtype=np.uint8)
    # uniform-k block (the GPU layer's layout)
    uni = [np.sort(rng.choice(32000, size=3200, replace=False)) for _ in range(16)]
    g["uni"] = np.stack(uni).astype(np.int32)
    g["uni_varint"] = np.frombuffer(SE.encode_index_sets(uni), dtype=np.uint8)
    np.savez_compressed(OUT / "serialize.npz", **g)
    print("wrote", OUT / "serialize.npz")


if __name__ == "__main__":
    main()
