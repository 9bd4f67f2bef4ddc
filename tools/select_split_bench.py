"""Fused selection vs key-range split (cluster size) at c2-like and c3-like shapes; split 0 =
the launcher's occupancy-based choice."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200 import ops  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for L, G, heads in ((32000, 260, (24, 12, 6, 3)), (131072, 1024, (16, 4, 2))):
        for H in heads:
            g = torch.Generator(device="cuda").manual_seed(0)
            qp = torch.randn((H, G, 16), device=dev, generator=g).to(torch.bfloat16)
            klr = torch.randn((H, L, 16), device=dev, generator=g).to(torch.bfloat16)
            k = int(0.1 * L)
            kp = torch.full((H,), k, dtype=torch.int32, device=dev)
            line = []
            for sp in (0, 1, 2, 4, 8):
                for _ in range(2):
                    ops.select_fused(qp, klr, kp, k, split=sp)
                ts = []
                for _ in range(9):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    ops.select_fused(qp, klr, kp, k, split=sp)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                line.append(f"s{sp}={sorted(ts)[4]:.3f}")
            print(f"L={L} H={H} tiles={H * ((G + 127) // 128)}: " + " ".join(line), flush=True)


if __name__ == "__main__":
    main()
