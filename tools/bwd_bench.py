"""Sparse backward alone at c2 (random sorted index lists, k = 3200): median of CUDA-event
timed launches (accumulators zeroed outside the timed region). DSV_LIB=<variant .so>."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200 import ops  # noqa: E402
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402
from paper_2502_07590_b200.grouping import build_groups  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    H, D, k = 24, 128, 3200
    plan = build_groups(TokenGrid(16, 40, 50), (8, 4, 4))
    L, G = plan.grid.size, plan.n_groups
    g = torch.Generator(device="cuda").manual_seed(0)
    idx = torch.stack([torch.randperm(L, device=dev, generator=g)[:k].sort().values for _ in range(H * G)])
    idx = idx.to(torch.int32).reshape(H, G, k)
    kp = torch.full((H,), k, dtype=torch.int32, device=dev)
    q, kk, v, do = (torch.randn((H, L, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
    rows, size = plan.tables(dev)
    o, lse = ops.sparse_fwd(q, kk, v, rows, size, idx, kp)
    dk = torch.zeros((H, L, D), device=dev)
    dv = torch.zeros_like(dk)
    ts = []
    for it in range(23):
        dk.zero_()
        dv.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ops.sparse_bwd(q, kk, v, o, do, lse, rows, size, idx, kp, None, dk, dv)
        b.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(a.elapsed_time(b))
    ts.sort()
    fl = 10 * H * L * k * D
    print(f"bwd median {ts[10]:.4f} ms min {ts[0]:.4f} ms  {fl / ts[10] / 1e9:.0f} TFLOP/s")


if __name__ == "__main__":
    main()
