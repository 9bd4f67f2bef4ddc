"""Hybrid head x selective-sequence CP (g_h = 2, g_s = 2) with world_size 4 on gloo.

cp.HybridExchange — the code the NCCL path runs — moves Q/K/V inside each SCP group
(HCP), gathers exactly the requested remote K/V rows between the ranks that hold the
same heads (SCP), and returns the outputs; the per-rank attention is the CPU oracle
(test injection). Outputs and every rank's byte ledger per phase must equal the
reference simulator's (tests/golden/cp_hybrid.npz from cpsim.run_hybrid_sparse_cp), for
both placements. The backward exchange (gradients of gathered rows back to their
owners) is checked as the adjoint of the forward gather.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN

PHASES = ("hcp_fwd", "scp_index_exchange", "scp_kv", "output_redistribute")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, placement, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2502_07590_b200.cp import HybridExchange

        g = np.load(GOLDEN / "cp_hybrid.npz")
        tag = placement.replace("-", "_")
        H, S, D = g["q"].shape
        chunk = S // world
        ptr, cols = g["ptr"], g["cols"]
        sets = [[cols[ptr[h * S + s]:ptr[h * S + s + 1]] for s in range(S)] for h in range(H)]
        rows = slice(rank * chunk, (rank + 1) * chunk)

        def run(dtype):
            ex = HybridExchange(H, S, g["assign"], 2, 2, placement)
            loc = [torch.from_numpy(g[n][:, rows].copy()).to(dtype) for n in ("q", "k", "v")]
            qs, ks, vs = (ex.hcp.to_heads(t) for t in loc)
            req = ex.requests_from_sets(sets)
            remote = ex.fetch_kv(ks, vs, req)
            return ex, qs, ks, vs, req, remote

        # ---- numerics (float64 payloads)
        ex, qs, ks, vs, req, remote = run(torch.float64)
        hp = len(ex.heads)
        kf = np.full((hp, S, D), np.nan)
        vf = np.full((hp, S, D), np.nan)
        kf[:, ex.span] = ks.numpy()
        vf[:, ex.span] = vs.numpy()
        for gp, per_head in req.items():
            for hi, r in enumerate(per_head):
                kf[hi, r] = remote[gp][hi][0].numpy()
                vf[hi, r] = remote[gp][hi][1].numpy()
        outs = []
        for hi, h in enumerate(ex.heads):
            o, _ = oracle.rows_attention_fwd(qs[hi].numpy(), kf[hi], vf[hi], [sets[h][x] for x in ex.span])
            outs.append(o)
        back = ex.hcp.to_tokens(torch.from_numpy(np.stack(outs)))
        np.testing.assert_allclose(back.numpy(), g[f"{tag}_out"][:, rows], atol=1e-10)
        # ---- adjoint: gradients of the gathered rows return to their owners
        dks = torch.zeros_like(ks)
        dvs = torch.zeros_like(vs)
        dk_rows = {gp: [torch.ones((len(r), D), dtype=torch.float64) for r in per]
                   for gp, per in req.items()}
        ex.return_grads(dk_rows, dk_rows, dks, dvs)
        # owner-side count of how many peers requested each of its rows, per head
        asked = np.zeros((hp, ex.span_len))
        for gp in range(ex.g_s):
            if gp == ex.grp:
                continue
            counts, ids = ex._served[gp]
            o = 0
            for hi, c in enumerate(counts):
                np.add.at(asked[hi], ex.local_at[ids[o:o + c].numpy()], 1.0)
                o += c
        np.testing.assert_array_equal(dks[:, :, 0].numpy(), asked)
        # ---- the device-vectorised exchange HybridDSV runs (requests_dev / fetch_kv_dev /
        # return_grads_dev): the same rows, the same adjoint, the same ledger
        def run_dev(dtype):
            ex = HybridExchange(H, S, g["assign"], 2, 2, placement)
            loc = [torch.from_numpy(g[n][:, rows].copy()).to(dtype) for n in ("q", "k", "v")]
            _, ks, vs = (ex.hcp.to_heads(t) for t in loc)
            mark = torch.zeros((len(ex.heads), S), dtype=torch.bool)
            for hi, h in enumerate(ex.heads):
                for x in ex.span:
                    mark[hi, torch.from_numpy(np.asarray(sets[h][x], dtype=np.int64))] = True
            need, cnt = ex.requests_dev(mark)
            return ex, ks, vs, need, cnt, ex.fetch_kv_dev(ks, vs, need, cnt)

        exd, ksd, vsd, need, cnt, got = run_dev(torch.float64)
        want = ~np.isnan(kf[:, :, 0])
        want[:, ex.span] = False
        nd = need.numpy()
        assert sorted(map(tuple, nd.tolist())) == sorted(map(tuple, np.argwhere(want).tolist()))
        np.testing.assert_array_equal(got[:, :D].numpy(), kf[nd[:, 0], nd[:, 1]])
        np.testing.assert_array_equal(got[:, D:].numpy(), vf[nd[:, 0], nd[:, 1]])
        dk_full = torch.zeros((hp, S, D), dtype=torch.float64)
        dk_full[need[:, 0], need[:, 1]] = 1.0
        dks_d = torch.zeros_like(ksd)

        def add_home(flat, a, b):
            dks_d.view(-1, D).index_add_(0, flat, a)
        exd.return_grads_dev(dk_full, dk_full, need, cnt, add_home)
        np.testing.assert_array_equal(dks_d[:, :, 0].numpy(), asked)
        exd2 = run_dev(torch.float16)[0]
        exd2.hcp.to_tokens(torch.zeros((len(exd2.heads), exd2.span_len, D), dtype=torch.float16))
        for ph in PHASES:
            assert exd2.ledger.sent.get(ph, 0) == g[f"{tag}_sent_{ph}"][rank], (ph, "sent", "dev")
            assert exd2.ledger.received.get(ph, 0) == g[f"{tag}_recv_{ph}"][rank], (ph, "recv", "dev")
        # ---- byte ledger == reference simulator ledger (2-byte elements)
        ex2, _, _, _, _, _ = run(torch.float16)
        ex2.hcp.to_tokens(torch.zeros((len(ex2.heads), ex2.span_len, D), dtype=torch.float16))
        for ph in PHASES:
            assert ex2.ledger.sent.get(ph, 0) == g[f"{tag}_sent_{ph}"][rank], (ph, "sent")
            assert ex2.ledger.received.get(ph, 0) == g[f"{tag}_recv_{ph}"][rank], (ph, "recv")
        q.put((rank, "ok"))
    except Exception as e:  # surface worker failures to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()[-1500:]))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("placement", ["hcp-first", "scp-first"])
def test_hybrid_exchange_gloo_world4(placement):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 4, port, placement, q)) for r in range(4)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = dict(q.get(timeout=5) for _ in range(4))
    assert results == {r: "ok" for r in range(4)}, results
    assert all(p.exitcode == 0 for p in procs)
