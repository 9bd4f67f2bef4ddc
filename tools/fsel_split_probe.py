"""Fused selection per key-range split at c2 head counts: time, fallback tiles (band misses
re-run by the multi-pass list mode) and band entries per (row, CTA).
python tools/fsel_split_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2502_07590_b200 import _lib, ops  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    L, G = 32000, 260
    k = 3200
    lib = _lib.load()
    print("max resident clusters per split:",
          {s: lib.dsv_select_fused_max_clusters(s) for s in range(1, 9)}, flush=True)
    for H in (24, 12, 6, 3, 2, 1):
        g = torch.Generator(device="cuda").manual_seed(0)
        qp = torch.randn((H, G, 16), device=dev, generator=g).to(torch.bfloat16)
        klr = torch.randn((H, L, 16), device=dev, generator=g).to(torch.bfloat16)
        kp = torch.full((H,), k, dtype=torch.int32, device=dev)
        for sp in (0, 2, 3, 4, 5, 6, 7, 8):
            for _ in range(2):
                ops.select_fused(qp, klr, kp, k, split=sp, mode="fast")
            ts = []
            for _ in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ops.select_fused(qp, klr, kp, k, split=sp, mode="fast")
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            fb = ops.select_fast_fallbacks(H, G, L, k, sp, dev)
            bs = ops.select_band_stats(H, G, L, k, sp, sp, dev) if sp else None
            print(f"H={H} split={sp}: {sorted(ts)[3]:.3f} ms fallback tiles {fb} band/CTA {bs}", flush=True)


if __name__ == "__main__":
    main()
