"""Fused K1b+K2 (select_fused.cu) vs unfused (tcgen05 GEMM scores + K2 top-k), timed with
CUDA events on the c2 / c3 / c5 selection shapes."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2502_07590_b200 import ops  # noqa: E402

SHAPES = {"c2": (24, 260, 32760, 3276), "c3": (16, 1024, 131072, 13108),
          "c5h2": (2, 4096, 524288, 52429)}


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for name in (sys.argv[1:] or SHAPES):
    H, G, L, k = SHAPES[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((H, G, 16), device="cuda", generator=g).to(torch.bfloat16)
    kl = torch.randn((H, L, 16), device="cuda", generator=g).to(torch.bfloat16)
    kc = torch.full((H,), k, dtype=torch.int32, device="cuda")
    idx = torch.empty((H * G, k), dtype=torch.int32, device="cuda")
    thr = torch.empty((H * G,), dtype=torch.float32, device="cuda")
    sc = torch.empty((H, G, L), dtype=torch.float32, device="cuda")
    t_g = timeit(lambda: ops.gemm_bf16(q, kl, torch.float32, out=sc))
    t_t = timeit(lambda: ops.topk_rows(sc.view(H * G, L), kc, G, k, out=(idx, thr)))
    line = f"{name}: unfused gemm {t_g:.3f} + topk {t_t:.3f} = {t_g + t_t:.3f} ms | fused"
    for s in (0, 1, 2, 3, 4):
        t = timeit(lambda: ops.select_fused(q, kl, kc, k, split=s, out=(idx, thr)))
        line += f" s{s}={t:.3f}"
    print(line, flush=True)
