"""Run each hot-path kernel once at the c2 shape (for ncu captures)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200 import ops
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.grouping import build_groups


def main(which):
    dev = torch.device("cuda:0")
    H, D, r, k = 24, 128, 16, 3200
    plan = build_groups(TokenGrid(16, 40, 50), (8, 4, 4))
    L, G = plan.grid.size, plan.n_groups
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn((L, H * D), device=dev, generator=g).to(torch.bfloat16)
    Wt = (torch.randn((2 * r * H, H * D), device=dev, generator=g) / math.sqrt(H * D)).to(torch.bfloat16)
    P = ops.project(X, Wt)
    qlr = P[:, : r * H].reshape(L, H, r)
    klr = P[:, r * H:].reshape(L, H, r).permute(1, 0, 2).contiguous()
    qp = qlr[plan.proxies_tensor(dev).long()].permute(1, 0, 2).contiguous()
    sc = ops.gemm_bf16(qp, klr, torch.float32).reshape(H * G, L)   # the layer's K1b path
    kp = torch.full((H,), k, dtype=torch.int32, device=dev)
    idx, _ = ops.topk_rows(sc, kp, G)
    ops.select_fused(qp, klr, kp, k)                                 # the layer's default (fused K1b+K2)
    idx = idx.reshape(H, G, k)
    q, kk, v, do = (torch.randn((H, L, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
    rows, size = plan.tables(dev)
    o, lse = ops.sparse_fwd(q, kk, v, rows, size, idx, kp)
    # as the layer runs it: dK / dV converted to bf16 in the kernel's tail
    dkdv = torch.empty((2, H, L, D), device=dev, dtype=torch.bfloat16)
    ops.sparse_bwd(q, kk, v, o, do, lse, rows, size, idx, kp, dkdv_out=dkdv)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main(sys.argv[1:] if len(sys.argv) > 1 else None)
