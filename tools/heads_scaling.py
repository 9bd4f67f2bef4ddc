"""One rank's share of c2 under head-parallel CP, on one GPU: the layer step (selection,
forward, backward) with 24 / 12 / 6 / 3 heads, per-stage CUDA-event times (median of 10
back-to-back steps). Shows the small-problem overheads (tile tails, selection fixed costs)
that separate N-GPU efficiency from linear. python tools/heads_scaling.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402
from paper_2502_07590_b200.layer import DSVAttentionLayer  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    D, r, L = 128, 16, 32000
    base = None
    for H in (24, 12, 6, 3):
        layer = DSVAttentionLayer(TokenGrid(16, 40, 50), H, D, r, (8, 4, 4), 0.9, dev)
        wt = layer.predictor_weights()
        g = torch.Generator(device=dev).manual_seed(0)
        x = torch.randn((L, H * D), device=dev, generator=g).to(torch.bfloat16)
        q, k, v, do = (torch.randn((H, L, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
        rows = []
        for it in range(13):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record()
            sel = layer.select(x, wt)
            e[1].record()
            out, lse = layer.forward(q, k, v, sel)
            e[2].record()
            layer.backward(q, k, v, out, lse, do, sel)
            e[3].record()
            rows.append(e)
        torch.cuda.synchronize()
        t = [sorted(r[i].elapsed_time(r[i + 1]) for r in rows[3:])[5] for i in range(3)]
        tot = sum(t)
        if base is None:
            base = tot
        print(f"H={H:2d}: select {t[0]:.3f} fwd {t[1]:.3f} bwd {t[2]:.3f} total {tot:.3f} ms "
              f"(linear share {base * H / 24:.3f}, efficiency {base * H / 24 / tot:.2f})", flush=True)


if __name__ == "__main__":
    main()
