"""Fused selection: single-pass (fast) vs multi-pass mode on the c2 / c3 shapes (CUDA events),
plus the fast mode's fallback tile count. python tools/fsel_modes.py [c2 c3 ...]"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2502_07590_b200 import ops  # noqa: E402

SHAPES = {"c2": (24, 260, 32000, 3200), "c3": (16, 1024, 131072, 13108),
          "c2h12": (12, 260, 32000, 3200), "c4h6": (6, 1024, 131072, 13108)}


def timeit(fn, n=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for name in (sys.argv[1:] or ["c2", "c3"]):
    H, G, L, k = SHAPES[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((H, G, 16), device="cuda", generator=g).to(torch.bfloat16)
    kl = torch.randn((H, L, 16), device="cuda", generator=g).to(torch.bfloat16)
    kc = torch.full((H,), k, dtype=torch.int32, device="cuda")
    out_f = (torch.empty((H * G, k), dtype=torch.int32, device="cuda"),
             torch.empty((H * G,), dtype=torch.float32, device="cuda"))
    out_m = (torch.empty_like(out_f[0]), torch.empty_like(out_f[1]))
    tf = timeit(lambda: ops.select_fused(q, kl, kc, k, out=out_f, mode="fast"))
    fb = ops.select_fast_fallbacks(H, G, L, k, 0, q.device)
    bs = ops.select_band_stats(H, G, L, k, 0, 2 if name.startswith("c2") else 1, q.device)
    tm = timeit(lambda: ops.select_fused(q, kl, kc, k, out=out_m, mode="multipass"))
    same = torch.equal(out_f[0], out_m[0]) and torch.equal(out_f[1], out_m[1])
    print(f"{name}: fast {tf:.3f} ms (fallback tiles {fb}, band/CTA mean,max {bs}) | multipass {tm:.3f} ms | identical {same}",
          flush=True)
