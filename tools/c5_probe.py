"""Long-sequence (c5, L=524288) diagnostic: bench-like allocations, one stage at a time,
index lists validated after each selection."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2502_07590_b200.grid import TokenGrid  # noqa: E402
from paper_2502_07590_b200.layer import DSVAttentionLayer  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 24
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
grid = TokenGrid(32, 128, 128)
L, D = grid.size, 128
layer = DSVAttentionLayer(grid, H, D, 16, (8, 4, 4), 0.9, dev)
wt = layer.predictor_weights(0)
g = torch.Generator(device=dev).manual_seed(1234)


def rnd(*s):
    return torch.randn(s, device=dev, generator=g).to(torch.bfloat16)


x, q, k, v, do = rnd(L, H * D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D)
dk = torch.zeros((H, L, D), device=dev, dtype=torch.float32)
dv = torch.zeros_like(dk)


def chk(name):
    torch.cuda.synchronize()
    print("ok", name, flush=True)


print("ptrs GB", [round(t.data_ptr() / 2**30, 2) for t in (x, q, k, v, do, dk, dv)], flush=True)
for s in range(steps):
    sel = layer.select(x, wt)
    chk(f"select {s}")
    idx = sel.idx
    lo, hi = int(idx.min()), int(idx.max())
    mono = bool((idx[:, :, 1:] > idx[:, :, :-1]).all())
    bad = ((idx < 0) | (idx >= L)).flatten(0, 1).any(dim=1).nonzero().flatten()
    print(f"idx range [{lo}, {hi}] ascending={mono} bad_rows={bad.numel()} first={bad[:8].tolist()}",
          flush=True)
    print("idx ptr GB", round(idx.data_ptr() / 2**30, 2), flush=True)
    out, lse = layer.forward(q, k, v, sel)
    chk(f"fwd {s}")
    layer.backward(q, k, v, out, lse, do, sel, dk, dv)
    chk(f"bwd {s}")
print("mem GB", torch.cuda.max_memory_allocated() / 1e9)
