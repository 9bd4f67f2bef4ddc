"""One fused selection launch (for ncu): python tools/fsel_once.py H G L k split"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2502_07590_b200 import ops  # noqa: E402

H, G, L, k, s = (int(x) for x in sys.argv[1:6])
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((H, G, 16), device="cuda", generator=g).to(torch.bfloat16)
kl = torch.randn((H, L, 16), device="cuda", generator=g).to(torch.bfloat16)
kc = torch.full((H,), k, dtype=torch.int32, device="cuda")
for _ in range(2):
    idx, thr = ops.select_fused(q, kl, kc, k, split=s)
torch.cuda.synchronize()
print("ok")
