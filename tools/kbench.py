"""Per-kernel timing at the BASELINE c2 shape (L=32000 = 16x40x50, H=24, d=128, k=3200).

CUDA events on the launching stream, warm-up first; prints one line per kernel.
"""
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2502_07590_b200 import ops
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.grouping import build_groups


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(iters):
        fn()
    en.record()
    torch.cuda.synchronize()
    return st.elapsed_time(en) / iters


def main():
    dev = torch.device("cuda:0")
    H, D, r = 24, 128, 16
    grid = TokenGrid(16, 40, 50)
    L = grid.size
    k = 3200
    plan = build_groups(grid, (8, 4, 4))
    G = plan.n_groups
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn((L, H * D), device=dev, generator=g).to(torch.bfloat16)
    Wt = (torch.randn((2 * r * H, H * D), device=dev, generator=g) / math.sqrt(H * D)).to(torch.bfloat16)
    t = timeit(lambda: ops.project(X, Wt))
    fl = 2 * L * H * D * 2 * r * H
    print(f"project   {t:8.3f} ms  {fl / t / 1e9:8.1f} TFLOP/s")
    P = ops.project(X, Wt)
    qlr = P[:, : r * H].reshape(L, H, r)
    klr = P[:, r * H:].reshape(L, H, r).permute(1, 0, 2).contiguous()   # [H, L, r]
    prox = plan.proxies_tensor(dev).long()
    qp = qlr[prox].permute(1, 0, 2).contiguous()                      # [H, G, r]
    t = timeit(lambda: ops.gemm_bf16(qp, klr, torch.float32))
    by = H * G * L * 4
    print(f"scores_tc {t:8.3f} ms  {by / t / 1e6:8.1f} GB/s (write)")
    t = timeit(lambda: ops.proxy_scores(qp, klr))
    print(f"scores_t  {t:8.3f} ms  {by / t / 1e6:8.1f} GB/s (write)")
    ref = ops.gemm_bf16(qp, klr, torch.float32)
    print("proxy_scores max|diff| vs gemm:", float((ops.proxy_scores(qp, klr) - ref).abs().max()))
    t = timeit(lambda: ops.scores_f32(qp, klr))
    print(f"scores_f32{t:8.3f} ms  {by / t / 1e6:8.1f} GB/s (write)")
    sc = ops.gemm_bf16(qp, klr, torch.float32).reshape(H * G, L)
    kp = torch.full((H,), k, dtype=torch.int32, device=dev)
    t = timeit(lambda: ops.topk_rows(sc, kp, G))
    by = H * G * (L * 4 + k * 4 + 4)
    print(f"topk      {t:8.3f} ms  {by / t / 1e6:8.1f} GB/s")
    idx, _ = ops.topk_rows(sc, kp, G)
    idx = idx.reshape(H, G, k)
    q, kk, v, do = (torch.randn((H, L, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
    rows, size = plan.tables(dev)
    fl_f = 4 * L * k * D * H
    t = timeit(lambda: ops.sparse_fwd(q, kk, v, rows, size, idx, kp))
    print(f"fwd       {t:8.3f} ms  {fl_f / t / 1e9:8.1f} TFLOP/s")
    o, lse = ops.sparse_fwd(q, kk, v, rows, size, idx, kp)
    dk = torch.zeros((H, L, D), device=dev, dtype=torch.float32)
    dv = torch.zeros_like(dk)
    t = timeit(lambda: ops.sparse_bwd(q, kk, v, o, do, lse, rows, size, idx, kp, dk_acc=dk, dv_acc=dv))
    print(f"bwd       {t:8.3f} ms  {2.5 * fl_f / t / 1e9:8.1f} TFLOP/s")
    # index-set wire format: varint-delta encoding of the layer's critical sets on device
    from paper_2502_07590_b200 import serialize as SZ
    flat = idx.reshape(H * G, k)
    enc = SZ.encode_device(flat)
    t = timeit(lambda: SZ.encode_device(flat), iters=5, warm=1)
    print(f"varint    {t:8.3f} ms  {flat.numel() * 4 / 1e6:.0f} MB int32 -> {enc.numel() / 1e6:.0f} MB encoded")
    # sampled sparsity profiler (factor 16: 2000 rows per head scored against all keys)
    from paper_2502_07590_b200 import profiler as PF
    cfg = PF.SampleConfig(factor=16)
    t = timeit(lambda: PF.measure_block_sparsity(list(q), list(kk), 0.9, cfg), iters=3, warm=1)
    print(f"profiler  {t:8.3f} ms  (24 heads x 2000 sampled rows x {L} keys, theta 0.9)")
    # predictor training step for one head: X [L, H*D], 2000 sampled rows, fp32 target [2000, L]
    from paper_2502_07590_b200 import predictor as PR
    prm = PR.PredictorParams.initialize(H * D, r, seed=0)
    xs = X.double()
    rws = PF.sample_queries(L, cfg)
    tgt = torch.randn((rws.size, L), device=dev, generator=g)
    t = timeit(lambda: PR.train_step(prm, xs, tgt, rows=rws), iters=3, warm=1)
    print(f"predictor {t:8.3f} ms  (one head: train_step, R=2000 rows x {L} keys, d={H * D}, r={r})")


if __name__ == "__main__":
    main()
