"""HCP on N GPUs vs the single-GPU layer on the same inputs (torchrun, NCCL).

usage: torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/cp_check.py [--skewed] [--hybrid]
                [--gs=G] [--dense=M] [--transport=peer|all_to_all] [--voxel=t,h,w]
(--hybrid: g_h = N/G head groups x g_s = G (default 2) selective-sequence groups, HybridDSV;
 --dense=M: the first M heads are dense residual heads, run by the ring KV pass)
Every rank builds the same global inputs (seeded), keeps its L/N token chunk, runs
HeadParallelDSV.step; the chunks of O, dQ, dK, dV are gathered and compared with
DSVAttentionLayer.step on rank 0, and the exchange ledger with hcp_comm.
"""

import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2502_07590_b200 import cpmodel  # noqa: E402
from paper_2502_07590_b200.cp import HeadParallelDSV, HybridDSV  # noqa: E402
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402
from paper_2502_07590_b200.layer import DSVAttentionLayer  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    hybrid = "--hybrid" in sys.argv
    gs = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--gs=")), 2))
    # hybrid: every SCP span must hold whole voxel groups (8 frames deep)
    grid = TokenGrid(8 * gs, 16, 16) if hybrid else TokenGrid(8, 16, 16)
    # --voxel=t,h,w: ladder shapes of more than 128 queries (128-query tiles sharing an index row)
    voxel = tuple(int(v) for v in next((a.split("=")[1] for a in sys.argv if a.startswith("--voxel=")),
                                       "8,4,4").split(","))
    H, D, r = 8, 128, 16
    L = grid.size
    sp = np.linspace(0.5, 0.95, H) if "--skewed" in sys.argv else np.full(H, 0.9)
    n_dense = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--dense=")), 0))
    sp[:n_dense] = 0.0                      # dense residual heads (k = L on one GPU)
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn((L, H * D), generator=g).to(torch.bfloat16).to(dev)
    q, k, v, do = (torch.randn((H, L, D), generator=g).to(torch.bfloat16).to(dev) for _ in range(4))
    wt = (torch.randn((2 * H * r, H * D), generator=g) / math.sqrt(H * D)).to(torch.bfloat16).to(dev)
    chunk = L // world
    sl = slice(rank * chunk, (rank + 1) * chunk)
    if hybrid:
        cp = HybridDSV(grid, H, D, r, voxel, sp, world // gs, gs, balanced=True, device=dev)
    else:
        tr = next((a.split("=")[1] for a in sys.argv if a.startswith("--transport=")), "auto")
        cp = HeadParallelDSV(grid, H, D, r, voxel, sp, balanced=True, device=dev, transport=tr)
    outs = cp.step(x[sl].contiguous(), wt, *(t[:, sl].contiguous() for t in (q, k, v, do)))
    gathered = []
    for t in outs:
        buf = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(buf, t.contiguous())
        gathered.append(torch.cat(buf, dim=1))
    ok = True
    if rank == 0:
        ref = DSVAttentionLayer(grid, H, D, r, voxel, sp, dev).step(x, wt, q, k, v, do)
        for name, a, b in zip(("out", "dq", "dk", "dv"), gathered, ref):
            err = (a.float() - b.float()).abs().max().item()
            rel = ((a.float() - b.float()).norm() / b.float().norm()).item()
            print(f"{name}: max|diff| {err:.3g} rel {rel:.3g}")
            ok &= rel < 1e-2
        print("assignment", cp.assignment.tolist())
    led = cp.ex.ledger
    if hybrid:
        print(f"rank {rank}: ledger sent {led.sent} received {led.received}")
        if getattr(cp, "scp", None) is not None:
            print(f"rank {rank}: SCP rows pulled over NVLink {int(cp.scp.pulled.item())}")
    else:
        got = max(led.sent["hcp_fwd"], led.received["hcp_fwd"])
        # one packed exchange of Q|K|V|Q_lr|K_lr: 3 D + 2 r columns per token
        expect_qkv = cpmodel.hcp_comm(H, len(cp.ex.my_heads), L, D, world, 2) * 3 / 4 * (3 * D + 2 * r) / (3 * D)
        print(f"rank {rank}: hcp_fwd bytes {got} (closed form for the packed payload {expect_qkv:.0f})")
    ok_t = torch.tensor([int(ok)], device=dev)
    dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    if rank == 0:
        print("CP CHECK", "PASS" if ok_t.item() else "FAIL")
    sys.exit(0 if ok_t.item() else 1)


if __name__ == "__main__":
    main()
