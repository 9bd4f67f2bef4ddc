"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the reference package `dynsparse` from /root/reference/pkg/src and
writes small .npz fixtures next to this file. The GPU box never needs
/root/reference: tests only read the committed fixtures.

Cases pin every hot-path function the oracle restates:
  selection  streaming_topk / twopass_select (random, heavy integer ties, given
             score matrices with +-0.0 ties via streaming_topk(S, I)), k_from_sparsity
  attention  full_attention, sparse_attention (uniform and ragged sets)
  grouping   build_groups members / proxies, grouped_sparse_attention
  backward   the trainer's own autograd path `_Block.attention(x, idx)`
             (trainer.py:104-118) with an identity qkv projection
  cp         balance_heads / hcp_comm / scp_comm / solve_hybrid and the cpsim
             ledger for head-parallel configurations
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    import torch

    from dynsparse import attention as A
    from dynsparse import cpmodel as CM
    from dynsparse import cpsim as CS
    from dynsparse import grouping as GR
    from dynsparse import selection as SE
    from dynsparse.grid import TokenGrid
    from dynsparse.trainer import ToyDiTConfig, _Block

    rng = np.random.default_rng(2025)

    # ------------------------------------------------------------ selection
    sel = {}
    q = rng.standard_normal((40, 6))
    k = rng.standard_normal((70, 6))
    r = SE.streaming_topk(q, k, 9)
    sel["rand_q"], sel["rand_k"], sel["rand_idx"], sel["rand_thr"] = q, k, r.indices, r.thresholds
    sel["rand_idx_twopass"] = SE.twopass_select(q, k, 9).indices
    qi = rng.integers(-4, 5, size=(64, 16)).astype(np.float64)
    ki = rng.integers(-4, 5, size=(300, 16)).astype(np.float64)
    r = SE.streaming_topk(qi, ki, 30)
    sel["ties_q"], sel["ties_k"], sel["ties_idx"], sel["ties_thr"] = qi, ki, r.indices, r.thresholds
    sel["ties_idx_twopass"] = SE.twopass_select(qi, ki, 30).indices
    # given score matrices (fp32 values, many ties, signed zeros): streaming_topk(S, I) == top-k of S
    vals = np.array([-0.0, 0.0, 1.0, -1.0, 0.5, 2.0, -3.0], dtype=np.float32)
    S = vals[rng.integers(0, vals.size, size=(32, 500))].astype(np.float64)
    S[:8] = rng.standard_normal((8, 500)).astype(np.float32)
    for kk in (1, 7, 120, 499, 500):
        rr = SE.streaming_topk(S, np.eye(500), kk)
        sel[f"given_idx_{kk}"], sel[f"given_thr_{kk}"] = rr.indices, rr.thresholds
    sel["given_scores"] = S.astype(np.float32)
    ks = [(0.9, 1000), (0.0, 7), (0.999, 100), (0.9, 4096), (0.9, 32000), (0.9, 131072),
          (0.9, 524288), (0.5, 131072), (0.95, 131072), (0.37, 12345)]
    sel["kfs_args"] = np.array(ks, dtype=np.float64)
    sel["kfs_k"] = np.array([SE.k_from_sparsity(s, n) for s, n in ks], dtype=np.int64)
    np.savez_compressed(OUT / "selection.npz", **sel)

    # ------------------------------------------------------------ attention
    att = {}
    q, k, v = (rng.standard_normal((12, 4)) for _ in range(3))
    att["q"], att["k"], att["v"] = q, k, v
    att["full"] = A.full_attention(q, k, v)
    uni = [np.sort(rng.choice(12, 5, replace=False)) for _ in range(12)]
    att["uni_idx"] = np.stack(uni)
    att["uni_out"] = A.sparse_attention(q, k, v, A.CriticalIndexSet(uni))
    rag = [np.sort(rng.choice(12, int(rng.integers(1, 13)), replace=False)) for _ in range(12)]
    att["rag_ptr"] = np.concatenate([[0], np.cumsum([len(x) for x in rag])])
    att["rag_cols"] = np.concatenate(rag)
    att["rag_out"] = A.sparse_attention(q, k, v, A.CriticalIndexSet(rag))
    np.savez_compressed(OUT / "attention.npz", **att)

    # ------------------------------------------------------------ grouping
    grp = {}
    cases = [((4, 4, 4), (2, 2, 2)), ((5, 4, 4), (2, 2, 2)), ((5, 6, 7), (2, 3, 4)),
             ((16, 40, 50), (8, 4, 4)), ((3, 3, 3), (3, 3, 3)), ((2, 3, 2), (1, 1, 1))]
    for i, (g, d) in enumerate(cases):
        plan = GR.build_groups(TokenGrid(*g), d)
        grp[f"c{i}_grid"], grp[f"c{i}_dims"] = np.array(g), np.array(d)
        grp[f"c{i}_proxies"] = plan.proxies
        grp[f"c{i}_sizes"] = np.array([m.size for m in plan.members])
        grp[f"c{i}_members"] = np.concatenate(plan.members)
    grid = TokenGrid(2, 4, 4)
    plan = GR.build_groups(grid, (2, 2, 2))
    qg, kg, vg = (rng.standard_normal((grid.size, 8)) for _ in range(3))
    sets = [np.sort(rng.choice(grid.size, int(rng.integers(3, 20)), replace=False))
            for _ in range(plan.n_groups)]
    grp["ga_q"], grp["ga_k"], grp["ga_v"] = qg, kg, vg
    grp["ga_ptr"] = np.concatenate([[0], np.cumsum([len(x) for x in sets])])
    grp["ga_cols"] = np.concatenate(sets)
    grp["ga_out"] = GR.grouped_sparse_attention(qg, kg, vg, plan, sets)
    np.savez_compressed(OUT / "grouping.npz", **grp)

    # ------------------------------------------------------------ backward (trainer autograd)
    bw = {}
    torch.manual_seed(0)
    H, dk, S, kk, B = 2, 8, 24, 6, 2
    cfg = ToyDiTConfig(heads=H, d_k=dk, hidden=3 * H * dk, d_lr=4)
    blk = _Block(cfg).double()
    with torch.no_grad():
        blk.qkv.weight.copy_(torch.eye(3 * H * dk, dtype=torch.float64))
        blk.qkv.bias.zero_()
    x = torch.randn(B, S, 3 * H * dk, dtype=torch.float64, requires_grad=True)
    idx = torch.stack([torch.stack([torch.sort(torch.randperm(S)[:kk]).values for _ in range(S)])
                       for _ in range(B)])
    out = blk.attention(x, idx)
    dout = torch.randn_like(out)
    (out * dout).sum().backward()
    bw["x"], bw["idx"], bw["out"], bw["dout"], bw["dx"] = (
        x.detach().numpy(), idx.numpy(), out.detach().numpy(), dout.numpy(), x.grad.numpy())
    bw["shape"] = np.array([B, S, H, dk])
    np.savez_compressed(OUT / "backward.npz", **bw)

    # ------------------------------------------------------------ cp planner + ledger
    cp = {}
    for i in range(20):
        h = int(rng.integers(2, 13))
        n = int(rng.integers(1, 5))
        loads = rng.uniform(0.5, 10.0, size=h)
        plan = CM.balance_heads(loads, n)
        cp[f"bh{i}_loads"], cp[f"bh{i}_n"] = loads, np.array(n)
        cp[f"bh{i}_comp"] = np.array(plan.comp_hcp)
        cp[f"bh{i}_assign"] = plan.assignment
    sp = 0.50 + 0.45 * np.arange(24) / 23
    rng.shuffle(sp)
    cp["c4_sparsities"] = sp
    for n in (2, 4, 8):
        plan = CM.balance_heads(CM.head_loads(sp, 131072, 128), n)
        cp[f"c4_n{n}_assign"], cp[f"c4_n{n}_comp"] = plan.assignment, np.array(plan.comp_hcp)
    hc = []
    for h_total, h_i, s, d, n, w in [(24, 3, 131072, 128, 8, 2), (16, 2, 131072, 128, 8, 2),
                                     (24, 12, 131072, 128, 2, 2), (4, 1, 64, 8, 4, 2)]:
        hc.append([h_total, h_i, s, d, n, w, CM.hcp_comm(h_total, h_i, s, d, n, w)])
    cp["hcp_comm"] = np.array(hc, dtype=np.float64)
    # cpsim head-parallel run: ledger + outputs
    h, s, d = 4, 64, 8
    q = rng.standard_normal((h, s, d))
    k = rng.standard_normal((h, s, d))
    v = rng.standard_normal((h, s, d))
    sets = []
    for hh in range(h):
        scores = A.attention_scores(q[hh], k[hh])
        sets.append(A.critical_kv_oracle(scores, 0.9).indices)
    sparsities = [1.0 - np.mean([x.size for x in per]) / s for per in sets]
    cluster = CM.ClusterSpec(n_devices=2, devices_per_node=2, intra_bw=1e9, inter_bw=1e8,
                             compute_rate=1e9, memory_cap=1e12, elem_width=2)
    plan = CM.balance_heads(CM.head_loads(sparsities, s, d), 2)
    conf = CM.CPConfig(g_h=2, g_s=1, placement="hcp-first", plan=plan, objective=0.0,
                       per_device_comp=[], per_device_comm=[], per_device_mem=[])
    devs = CS.make_devices(q, k, v, cluster, conf)
    out, log = CS.run_hybrid_sparse_cp(devs, conf, cluster, sets)
    cp["sim_q"], cp["sim_k"], cp["sim_v"], cp["sim_out"] = q, k, v, out
    cp["sim_assign"] = plan.assignment
    cp["sim_sent_hcp"] = np.array([log.sent_by(r, "hcp_fwd") for r in range(2)])
    cp["sim_recv_hcp"] = np.array([log.received_by(r, "hcp_fwd") for r in range(2)])
    cp["sim_sent_out"] = np.array([log.sent_by(r, "output_redistribute") for r in range(2)])
    cp["sim_recv_out"] = np.array([log.received_by(r, "output_redistribute") for r in range(2)])
    ptr = [0]
    cols = []
    for per in sets:
        for x_ in per:
            cols.append(np.asarray(x_))
            ptr.append(ptr[-1] + len(x_))
    cp["sim_ptr"], cp["sim_cols"] = np.array(ptr), np.concatenate(cols)
    np.savez_compressed(OUT / "cp.npz", **cp)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
