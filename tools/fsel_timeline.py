"""Pass timeline of the fused selection (CTA 0), from a -DDSV_FSEL_PROF=1 build:
DSV_LIB=build_var/lib_fprof.so python tools/fsel_timeline.py H G L k split"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2502_07590_b200 import _lib, ops  # noqa: E402

H, G, L, k, s = (int(x) for x in sys.argv[1:6])
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((H, G, 16), device="cuda", generator=g).to(torch.bfloat16)
kl = torch.randn((H, L, 16), device="cuda", generator=g).to(torch.bfloat16)
kc = torch.full((H,), k, dtype=torch.int32, device="cuda")
for _ in range(3):
    ops.select_fused(q, kl, kc, k, split=s)
torch.cuda.synchronize()
buf = np.zeros((64, 8), dtype=np.uint64)
n = _lib.load().dsv_debug_select_timeline(ctypes.c_void_p(buf.ctypes.data), buf.nbytes)
t0 = buf[0, 0]
names = ["start", "first", "tiles_done", "partials", "syncA", "final", "syncB", "next"]
for p in range(64):
    if buf[p, 0] == 0 or buf[p, 0] < t0:
        break
    print(p, " ".join(f"{names[e]}={(int(buf[p, e]) - int(t0)) / 1e3:.1f}" for e in range(8)))
