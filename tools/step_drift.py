"""Per-step stage times over a long run of back-to-back c2 steps (eager, CUDA events on the
compute stream), to see whether the backward kernel drifts under sustained load.
python tools/step_drift.py [steps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402
from paper_2502_07590_b200.layer import DSVAttentionLayer  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    dev = torch.device("cuda:0")
    H, D, r, L = 24, 128, 16, 32000
    layer = DSVAttentionLayer(TokenGrid(16, 40, 50), H, D, r, (8, 4, 4), 0.9, dev)
    wt = layer.predictor_weights()
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((L, H * D), device=dev, generator=g).to(torch.bfloat16)
    q, k, v, do = (torch.randn((H, L, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(n)]
    for i in range(n):
        e = evs[i]
        e[0].record()
        sel = layer.select(x, wt)
        e[1].record()
        out, lse = layer.forward(q, k, v, sel)
        e[2].record()
        layer.backward(q, k, v, out, lse, do, sel, kernel_done=e[3])
        e[4].record()
    torch.cuda.synchronize()
    for i in range(n):
        e = evs[i]
        print(f"step {i:3d}: select {e[0].elapsed_time(e[1]):.3f} fwd {e[1].elapsed_time(e[2]):.3f} "
              f"bwd_kernel {e[2].elapsed_time(e[3]):.3f} convert {e[3].elapsed_time(e[4]):.3f} "
              f"total {e[0].elapsed_time(e[4]):.3f}")


if __name__ == "__main__":
    main()
