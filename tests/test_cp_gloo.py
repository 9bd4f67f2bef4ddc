"""Head-parallel CP protocol with world_size 2 on the gloo backend (CPU only).

The exchange layer (paper_2502_07590_b200.cp.HeadParallelExchange) is the same
code the NCCL path runs; here the per-rank attention is the CPU oracle (test
injection) so the whole Algorithm-1 HCP pipeline can be checked against the
reference simulator's outputs and byte ledger (tests/golden/cp.npz, produced by
cpsim.run_hybrid_sparse_cp with g_h = 2, g_s = 1).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2502_07590_b200 import cpmodel
        from paper_2502_07590_b200.cp import HeadParallelExchange

        g = np.load(GOLDEN / "cp.npz")
        H, S, D = g["sim_q"].shape
        chunk = S // world
        ex = HeadParallelExchange(H, S, g["sim_assign"])
        ptr, cols = g["sim_ptr"], g["sim_cols"]
        sets = [[cols[ptr[h * S + s]:ptr[h * S + s + 1]] for s in range(S)] for h in range(H)]
        # ---- round trip + numerical equivalence (float64 payloads)
        loc = [torch.from_numpy(g[f"sim_{n}"][:, rank * chunk:(rank + 1) * chunk].copy())
               for n in ("q", "k", "v")]
        mine = [ex.to_heads(t) for t in loc]
        for t, name in zip(mine, ("q", "k", "v")):
            np.testing.assert_array_equal(t.numpy(), g[f"sim_{name}"][ex.my_heads])
        outs = []
        for hi, h in enumerate(ex.my_heads):
            o, _ = oracle.rows_attention_fwd(mine[0][hi].numpy(), mine[1][hi].numpy(),
                                             mine[2][hi].numpy(), sets[h])
            outs.append(o)
        back = ex.to_tokens(torch.from_numpy(np.stack(outs)))
        np.testing.assert_allclose(back.numpy(), g["sim_out"][:, rank * chunk:(rank + 1) * chunk],
                                   atol=1e-10)
        # ---- byte ledger == reference simulator ledger == closed form (2-byte elements)
        ex2 = HeadParallelExchange(H, S, g["sim_assign"])
        for t in loc:
            ex2.to_heads(t.to(torch.float16))
        ex2.to_tokens(torch.zeros((len(ex2.my_heads), S, D), dtype=torch.float16))
        assert ex2.ledger.sent["hcp_fwd"] == g["sim_sent_hcp"][rank]
        assert ex2.ledger.received["hcp_fwd"] == g["sim_recv_hcp"][rank]
        assert ex2.ledger.sent["output_redistribute"] == g["sim_sent_out"][rank]
        assert ex2.ledger.received["output_redistribute"] == g["sim_recv_out"][rank]
        got = (max(ex2.ledger.sent["hcp_fwd"], ex2.ledger.received["hcp_fwd"])
               + max(ex2.ledger.sent["output_redistribute"], ex2.ledger.received["output_redistribute"]))
        assert got == cpmodel.hcp_comm(H, len(ex2.my_heads), S, D, world, 2)
        q.put((rank, "ok"))
    except Exception as e:  # surface worker failures to the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_hcp_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: "ok", 1: "ok"}, results
    assert all(p.exitcode == 0 for p in procs)


def test_plan_heads_balanced_vs_contiguous():
    from paper_2502_07590_b200.cp import plan_heads

    sp = np.linspace(0.5, 0.95, 8)
    a = plan_heads(sp, 1024, 64, 4, balanced=True)
    b = plan_heads(sp, 1024, 64, 4, balanced=False)
    assert sorted(np.bincount(b, minlength=4)) == [2, 2, 2, 2]
    from paper_2502_07590_b200 import cpmodel

    loads = cpmodel.head_loads(sp, 1024, 64)
    ca = max(loads[a == r].sum() for r in range(4))
    cb = max(loads[b == r].sum() for r in range(4))
    assert ca <= cb


def test_plan_heads_from_measured_profile():
    # measured per-head sparsity (profiler EMA) drives the re-balancing
    from paper_2502_07590_b200 import cpmodel
    from paper_2502_07590_b200.cp import plan_heads, plan_heads_from_profile
    from paper_2502_07590_b200.profiler import SparsityProfile

    prof = SparsityProfile(alpha=0.5)
    rng = np.random.default_rng(3)
    for it in range(4):
        prof.update_block(2, rng.uniform(0.5, 0.95, size=8), it)
    assign, sp = plan_heads_from_profile(prof, 2, 4096, 64, 4)
    np.testing.assert_array_equal(sp, prof.head_emas(2))
    np.testing.assert_array_equal(assign, plan_heads(sp, 4096, 64, 4))
    loads = cpmodel.head_loads(sp, 4096, 64)
    naive = plan_heads(sp, 4096, 64, 4, balanced=False)
    assert max(loads[assign == r].sum() for r in range(4)) <= max(loads[naive == r].sum() for r in range(4))
    with pytest.raises(ValueError):
        plan_heads_from_profile(prof, 7, 4096, 64, 4)


def _worker_no_heads(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_07590_b200.cp import HeadParallelDSV
        from paper_2502_07590_b200.grid import TokenGrid

        try:
            HeadParallelDSV(TokenGrid(8, 4, 4), 1, 64, 16, (8, 4, 4), 0.9, device="cpu",
                            transport="all_to_all")
            q.put((rank, "no error"))
        except ValueError as e:
            q.put((rank, "ValueError" if "HybridDSV" in str(e) else repr(e)))
    finally:
        dist.destroy_process_group()


def test_head_parallel_fewer_heads_than_ranks_raises_on_every_rank():
    # one head over two ranks: both raise before any collective (none is left waiting)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_no_heads, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: "ValueError", 1: "ValueError"}, results
