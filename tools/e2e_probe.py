"""Timeline of HostPipeline at c2 with the D2H of each step's results: per-step compute
(start, end) and D2H (end) events, relative to the first copy. python tools/e2e_probe.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402
from paper_2502_07590_b200.layer import DSVAttentionLayer, HostPipeline  # noqa: E402


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
    pipe = HostPipeline(host, dev)
    marks = []

    def step(*b):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        out = layer.step(b[0], wt, *b[1:])
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        marks.append([e0, e1])
        return out

    for rep in range(2):
        marks.clear()
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in pipe.run(step, [host] * 6):
            e2 = torch.cuda.Event(enable_timing=True)
            e2.record(pipe.d2h)
            marks[-1].append(e2)
        pipe.drain()
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record()
        torch.cuda.synchronize()
        print(f"rep {rep}: {t0.elapsed_time(t1) / 6:.2f} ms/step")
        for i, (a, b, c) in enumerate(marks):
            print(f"  step {i}: compute {t0.elapsed_time(a):7.2f} .. {t0.elapsed_time(b):7.2f}  "
                  f"d2h done {t0.elapsed_time(c):7.2f}")


if __name__ == "__main__":
    main()
