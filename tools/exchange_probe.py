"""Timing of the HCP input-exchange pieces at c2 (torchrun, NCCL): device barrier, Q_lr/K_lr
copy, Q/K/V/dO copy, each alone on the compute stream (CUDA events, median of 20, max over
ranks). torchrun --nproc-per-node N tools/exchange_probe.py"""
import math
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.getcwd())
from paper_2502_07590_b200 import ops  # noqa: E402
from paper_2502_07590_b200.cp import HeadParallelDSV  # noqa: E402
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    H, D, r = 24, 128, 16
    grid = TokenGrid(16, 40, 50)
    L = grid.size
    cp = HeadParallelDSV(grid, H, D, r, (8, 4, 4), 0.9, device=dev)
    chunk = L // world
    g = torch.Generator(device=dev).manual_seed(rank)
    x = torch.randn((chunk, H * D), device=dev, generator=g).to(torch.bfloat16)
    q, k, v, do = (torch.randn((H, chunk, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
    wt = (torch.randn((2 * H * r, H * D), device=dev, generator=g) / math.sqrt(H * D)).to(torch.bfloat16)
    for _ in range(3):
        cp.step(x, wt, q, k, v, do)
    torch.cuda.synchronize()
    ex = cp.ex
    p = ops.project(x, wt)
    key = ("fo",) + tuple(t.data_ptr() for t in (q, k, v, do, p))
    low = ex._table(key + ("lr",), lambda: ex._lowrank_jobs(p))
    big = ex._table(key + ("big",), lambda: ex._head_jobs((("q", q), ("k", k), ("v", v), ("do", do))))
    sm = torch.cuda.get_device_properties(dev).multi_processor_count
    pieces = {
        "barrier": lambda: ex._barrier(),
        "lowrank copy (splits 16)": lambda: ops.copy_jobs(low, ex.splits),
        "QKVdO copy (1 CTA/SM grid)": lambda: ops.copy_jobs(big, max(1, -(-sm // big.shape[0]))),
        "QKVdO copy (splits 16)": lambda: ops.copy_jobs(big, 16),
        "projection": lambda: ops.project(x, wt),
    }
    res = {}
    for name, fn in pieces.items():
        ts = []
        for _ in range(20):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = torch.tensor([sorted(ts)[10]], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = t.item()
    if rank == 0:
        print(f"N={world}: " + " | ".join(f"{k} {v * 1e3:.1f} us" for k, v in res.items()), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
