"""Timeline of HostPipeline at c2: copy-stream and compute-stream events per step."""
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.layer import DSVAttentionLayer, HostPipeline


def main():
    dev = torch.device("cuda:0")
    H, D, r = 24, 128, 16
    grid = TokenGrid(16, 40, 50)
    L = grid.size
    layer = DSVAttentionLayer(grid, H, D, r, (8, 4, 4), 0.9, dev)
    wt = layer.predictor_weights()
    g = torch.Generator().manual_seed(0)
    host = [torch.randn(s, generator=g).to(torch.bfloat16).pin_memory()
            for s in ((L, H * D), (H, L, D), (H, L, D), (H, L, D), (H, L, D))]
    dk = torch.zeros((H, L, D), device=dev)
    dv = torch.zeros_like(dk)
    pipe = HostPipeline(host, dev)
    marks = []

    def step(*b):
        e0 = torch.cuda.Event(enable_timing=True); e0.record()
        out = layer.step(b[0], wt, *b[1:], dk_acc=dk, dv_acc=dv)
        e1 = torch.cuda.Event(enable_timing=True); e1.record()
        marks.append((e0, e1))
        return out

    for mode in ("pipe", "pipe"):
        marks.clear()
        t0 = torch.cuda.Event(enable_timing=True); t0.record()
        w0 = time.perf_counter()
        for out in pipe.run(step, [host] * 5):
            float(out[1].float().sum().item())
        t1 = torch.cuda.Event(enable_timing=True); t1.record()
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        print(f"{mode}: total {t0.elapsed_time(t1):.2f} ms (wall {1e3 * (w1 - w0):.2f}) for 5 steps")
        for i, (a, b) in enumerate(marks):
            print(f"  step {i}: start {t0.elapsed_time(a):7.2f}  end {t0.elapsed_time(b):7.2f}")
    # plain sequential copy then step
    bufs = pipe.bufs[0]
    t0 = torch.cuda.Event(enable_timing=True); t0.record()
    for _ in range(5):
        for s_, d_ in zip(host, bufs):
            d_.copy_(s_, non_blocking=True)
        out = layer.step(bufs[0], wt, *bufs[1:], dk_acc=dk, dv_acc=dv)
        float(out[1].float().sum().item())
    t1 = torch.cuda.Event(enable_timing=True); t1.record()
    torch.cuda.synchronize()
    print(f"sequential: {t0.elapsed_time(t1) / 5:.2f} ms/step")


if __name__ == "__main__":
    main()
