"""Phase timeline of the sparse forward at c2 (needs a -DDSV_FWD_PROF build via DSV_LIB).
Events: 0 S_j issue, 1 PV_j issue, 2 softmax sees S_j, 3 pass 1 done, 4 P_j ready, 5 K_j load, 6 V_j load."""
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
    q, kk, v = (torch.randn((H, L, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
    rows, size = plan.tables(dev)
    for _ in range(3):
        ops.sparse_fwd(q, kk, v, rows, size, idx, kp)
    torch.cuda.synchronize()
    buf = np.zeros((8, 32, 12), dtype=np.int64)
    n = _lib.load().dsv_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes)
    assert n == buf.nbytes
    names = ["S", "PV", "sm0", "sm1", "P", "loadK", "loadV"]
    t = buf[:, :, :7].astype(np.float64)
    for cta in range(1):
        t0 = t[cta, 0, 0]
        print(f"CTA {cta}:  j " + " ".join(f"{x:>7s}" for x in names))
        for j in range(0, 25):
            print(f"        {j:2d} " + " ".join(f"{x - t0:7.0f}" for x in t[cta, j]))
    tt = t[:, 2:24]
    per = lambda a, b: np.median(tt[:, :, b] - tt[:, :, a])
    print("median (cycles): period S_j->S_j+1", np.median(np.diff(t[:, 2:25, 0], axis=1)))
    print("  S issue -> softmax sees S", per(0, 2))
    print("  pass 1 (max)             ", per(2, 3))
    print("  pass 2 (exp, P)          ", per(3, 4))
    print("  P ready -> PV issue      ", per(4, 1))
    print("  load K_j -> S_j issue    ", per(5, 0))
    print("  load V_j -> PV_j issue   ", per(6, 1))
    tf = buf[:, 2:24, :].astype(np.float64)
    pf = lambda a, b: np.median(tf[:, :, b] - tf[:, :, a])
    print("  warp 0: sees S -> ld done", pf(2, 7), " max ->xch", pf(7, 8), " barrier", pf(8, 3),
          " P compute", pf(3, 9), " st wait+arrive", pf(9, 4))
    print("  softmax: P_j -> sees S_j+1", np.median(buf[:, 3:25, 2] - buf[:, 2:24, 4]))


if __name__ == "__main__":
    main()
