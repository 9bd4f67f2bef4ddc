"""Where the selective KV fetch (SCP) spends its time: torchrun --nproc-per-node 2
tools/scp_probe.py  (c2 shape, g_h = 1 x g_s = 2; host-timed with device syncs)."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2502_07590_b200.cp import HybridDSV  # noqa: E402
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    grid = TokenGrid(16, 40, 50)
    H, D, r = 24, 128, 16
    cp = HybridDSV(grid, H, D, r, (8, 4, 4), 0.9, 1, world, device=dev)
    ex, L = cp.ex, grid.size
    hs = len(cp.heads)
    g = torch.Generator(device=dev).manual_seed(rank)
    kl = torch.randn((hs, cp.span_len, D), device=dev, generator=g).to(torch.bfloat16)
    vl = torch.randn_like(kl)
    idx = torch.stack([torch.randperm(L, device=dev, generator=g)[:3200].sort().values
                       for _ in range(hs * cp.local.G)]).to(torch.int32).view(hs, cp.local.G, 3200)
    T = {}

    def t(name, fn):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        r_ = fn()
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
        return r_

    for it in range(4):
        if it == 1:
            T.clear()
        mark = t("mark", lambda: _mark(idx, cp.local.ks, L))
        need, cnt = t("requests_dev", lambda: ex.requests_dev(mark))
        got = t("fetch_kv_dev", lambda: ex.fetch_kv_dev(kl, vl, need, cnt))
        Kf = torch.empty((hs, L, D), dtype=torch.bfloat16, device=dev)
        flat = need[:, 0] * L + need[:, 1]
        t("index_copy", lambda: Kf.view(-1, D).index_copy_(0, flat, got[:, :D]))
    if rank == 0:
        print({k: round(v / 3, 3) for k, v in T.items()}, "rows", int(need.shape[0]))
    dist.destroy_process_group()


def _mark(idx, ks, L):
    hs = idx.shape[0]
    mark = torch.zeros((hs, L), dtype=torch.bool, device=idx.device)
    for hi, kh in enumerate(ks):
        mark[hi].index_fill_(0, idx[hi, :, :kh].reshape(-1).long(), True)
    return mark


if __name__ == "__main__":
    main()
