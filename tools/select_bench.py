"""Selection (K1b + K2) fused vs unfused across head counts / lengths: median CUDA-event
time of DSVAttentionLayer.select_from_lowrank. usage: python tools/select_bench.py"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402
from paper_2502_07590_b200.layer import DSVAttentionLayer  # noqa: E402


def timed(fn, n=15):
    for _ in range(3):
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
    dev = torch.device("cuda:0")
    for dims, heads in (((16, 40, 50), (24, 12, 6, 3)), ((32, 64, 64), (16, 8, 4, 2))):
        grid = TokenGrid(*dims)
        L = grid.size
        for H in heads:
            layer = DSVAttentionLayer(grid, H, 128, 16, (8, 4, 4), 0.9, dev)
            g = torch.Generator(device="cuda").manual_seed(0)
            qlr = torch.randn((H, L, 16), device=dev, generator=g).to(torch.bfloat16)
            klr = torch.randn((H, L, 16), device=dev, generator=g).to(torch.bfloat16)
            res = {}
            for mode in ("1", "0"):
                os.environ["DSV_FUSED_SELECT"] = mode
                res[mode] = timed(lambda: layer.select_from_lowrank(qlr, klr))
            tiles = H * ((layer.G + 127) // 128)
            print(f"L={L} H={H} G={layer.G} tiles={tiles}: fused {res['1']:.3f} ms  unfused {res['0']:.3f} ms",
                  flush=True)


if __name__ == "__main__":
    main()
