"""One fused selection call at a shape (for ncu launch lists):
python tools/fsel_once.py H G L k [fast|multipass] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2502_07590_b200 import ops  # noqa: E402

H, G, L, k = (int(x) for x in sys.argv[1:5])
mode = sys.argv[5] if len(sys.argv) > 5 else "fast"
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 2
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((H, G, 16), device="cuda", generator=g).to(torch.bfloat16)
kl = torch.randn((H, L, 16), device="cuda", generator=g).to(torch.bfloat16)
kc = torch.full((H,), k, dtype=torch.int32, device="cuda")
for _ in range(reps):
    ops.select_fused(q, kl, kc, k, mode=mode)
torch.cuda.synchronize()
print("fallback tiles", ops.select_fast_fallbacks(H, G, L, k, 0, q.device))
