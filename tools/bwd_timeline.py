"""Phase timeline of the sparse backward at c2 (needs a -DDSV_BWD_PROF build via DSV_LIB).

usage: DSV_LIB=paper_2502_07590_b200/libdsv_prof.so python tools/bwd_timeline.py
Events (clock64 per CTA): 0 V issue, 1 K issue, 2 A start (MMA), 3 C start (MMA),
4 B start (workers), 5 B end, 6 C' start, 7 C' end, 8 scatter dV start,
9 scatter dK start, 10 scatter end.
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200 import _lib, ops
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.grouping import build_groups


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
    for _ in range(3):
        ops.sparse_bwd(q, kk, v, o, do, lse, rows, size, idx, kp)
    torch.cuda.synchronize()
    buf = np.zeros((8, 32, 12), dtype=np.int64)
    n = _lib.load().dsv_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes)
    assert n == buf.nbytes, n
    names = ["Viss", "Kiss", "A", "C", "B0", "B1", "C'0", "C'1", "scV", "scK", "scE"]
    for cta in range(2):
        t = buf[cta, :, :11].astype(np.float64)
        t0 = t[0, 2]
        print(f"CTA {cta} (cycles rel. to A_0):")
        print("  j  " + " ".join(f"{x:>7s}" for x in names))
        for j in range(0, 25, 3):
            print(f" {j:2d}  " + " ".join(f"{x - t0:7.0f}" for x in t[j]))
    t = buf[:, 2:24, :11].astype(np.float64)
    per = lambda a, b: np.median(t[:, :, b] - t[:, :, a])
    print("median over CTAs 0-7, blocks 2-23 (cycles):")
    print("  period A_j -> A_j+1      ", np.median(np.diff(buf[:, 2:25, 2], axis=1)))
    print("  A start -> B start (MMA A)", per(2, 4))
    print("  B start -> B end (workers)", per(4, 5))
    print("  B end -> C start          ", per(5, 3))
    print("  C start -> C' start (MMA C)", per(3, 6))
    print("  C' start -> C' end        ", per(6, 7))
    print("  C' end -> next A start    ", np.median(buf[:, 3:25, 2] - buf[:, 2:24, 7]))
    print("  scatter dV (scV -> scK)   ", per(8, 9))
    print("  scatter dK (scK -> scE)   ", per(9, 10))
    print("  K issue -> A start         ", per(1, 2))
    print("  V issue -> A start         ", per(0, 2))


if __name__ == "__main__":
    main()
