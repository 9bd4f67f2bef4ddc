"""Sparse forward + backward alone at a given shape (random sorted index lists): median of
CUDA-event timed launches. usage: python tools/attn_bench.py T Hgt W H k   (grid T x Hgt x W)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200 import ops  # noqa: E402
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402
from paper_2502_07590_b200.grouping import build_groups  # noqa: E402


def timed(fn, n=9):
    fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[n // 2]


def main():
    T, Hg, W, H, k = (int(a) for a in sys.argv[1:6])
    dev = torch.device("cuda:0")
    plan = build_groups(TokenGrid(T, Hg, W), (8, 4, 4))
    L, G, D = plan.grid.size, plan.n_groups, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    idx = torch.stack([torch.randperm(L, device=dev, generator=g)[:k].sort().values for _ in range(H * G)])
    idx = idx.to(torch.int32).reshape(H, G, k)
    kp = torch.full((H,), k, dtype=torch.int32, device=dev)
    q, kk, v, do = (torch.randn((H, L, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
    rows, size = plan.tables(dev)
    o, lse = ops.sparse_fwd(q, kk, v, rows, size, idx, kp)
    dk = torch.zeros((H, L, D), device=dev)
    dv = torch.zeros_like(dk)
    tf = timed(lambda: ops.sparse_fwd(q, kk, v, rows, size, idx, kp))
    tb = timed(lambda: ops.sparse_bwd(q, kk, v, o, do, lse, rows, size, idx, kp, None, dk, dv))
    print(f"L={L} H={H} G={G} k={k}: fwd {tf:.3f} ms  bwd {tb:.3f} ms")


if __name__ == "__main__":
    main()
