"""The context-parallel layers on one B200 inside a world-1 NCCL process group.

The multi-GPU checks (tools/cp_check.py: HCP, hybrid, ring, overlap — bit-exact against the
one-GPU layer at 2 and 4 GPUs) need several GPUs; this runs the same code paths in the
single-GPU tier: HeadParallelDSV over both transports (peer memory and all-to-all) and
HybridDSV with dense residual heads (ring KV pass, n = 1) next to sparse heads, each
against DSVAttentionLayer.step on the same inputs. Forward outputs are deterministic
(equal); gradients differ only by the order of the fp32 atomic adds (rel-L2 <= 1e-2).
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.layer import DSVAttentionLayer

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def pg(cuda):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(cuda)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    yield
    dist.destroy_process_group()


def _inputs(grid, H, D, r, dev, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    L = grid.size
    x = torch.randn((L, H * D), generator=g).to(torch.bfloat16).to(dev)
    q, k, v, do = (torch.randn((H, L, D), generator=g).to(torch.bfloat16).to(dev) for _ in range(4))
    wt = (torch.randn((2 * H * r, H * D), generator=g) / math.sqrt(H * D)).to(torch.bfloat16).to(dev)
    return x, wt, q, k, v, do


def _rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("transport", ["peer", "all_to_all"])
def test_head_parallel_world1_matches_layer(cuda, pg, transport):
    from paper_2502_07590_b200.cp import HeadParallelDSV

    grid, H, D, r = TokenGrid(8, 16, 16), 4, 128, 16
    sp = np.array([0.5, 0.75, 0.9, 0.95])
    x, wt, q, k, v, do = _inputs(grid, H, D, r, cuda)
    cp = HeadParallelDSV(grid, H, D, r, (8, 4, 4), sp, device=cuda, transport=transport)
    got = [t.clone() for t in cp.step(x, wt, q, k, v, do)]
    ref = DSVAttentionLayer(grid, H, D, r, (8, 4, 4), sp, cuda).step(x, wt, q, k, v, do)
    torch.cuda.synchronize()
    assert torch.equal(got[0], ref[0])
    for a, b in zip(got[1:], ref[1:]):
        assert _rel(a, b) <= 1e-2


def test_hybrid_with_dense_heads_world1_matches_layer(cuda, pg):
    from paper_2502_07590_b200.cp import HybridDSV

    grid, H, D, r = TokenGrid(8, 16, 16), 4, 128, 16
    sp = np.array([0.0, 0.9, 0.0, 0.75])          # heads 0 and 2 dense: ring KV pass (n = 1)
    x, wt, q, k, v, do = _inputs(grid, H, D, r, cuda, seed=1)
    cp = HybridDSV(grid, H, D, r, (8, 4, 4), sp, 1, 1, device=cuda)
    assert sorted(int(cp.heads[i]) for i in cp.dloc) == [0, 2]
    got = [t.clone() for t in cp.step(x, wt, q, k, v, do)]
    ref = DSVAttentionLayer(grid, H, D, r, (8, 4, 4), sp, cuda).step(x, wt, q, k, v, do)
    torch.cuda.synchronize()
    for a, b in zip(got, ref):
        assert _rel(a, b) <= 1e-2
    w = cp.work()
    L = grid.size
    assert w["fwd_flops"] >= 2 * 4 * L * L * D          # the two dense heads at least


def test_measured_sparsity_drives_the_head_plan(cuda, pg):
    # profiler on the GPU -> SparsityProfile EMA -> balance_heads plan -> HCP layer
    from paper_2502_07590_b200.cp import HeadParallelDSV, plan_heads_from_profile
    from paper_2502_07590_b200.profiler import SampleConfig, SparsityProfile, measure_block_sparsity

    grid, H, D, r = TokenGrid(8, 16, 16), 4, 128, 16
    x, wt, q, k, v, do = _inputs(grid, H, D, r, cuda, seed=2)
    q = q * torch.tensor([0.5, 1.0, 2.0, 4.0], device=cuda, dtype=torch.bfloat16)[:, None, None]
    samples = measure_block_sparsity(list(q), list(k), 0.9, SampleConfig(factor=16))
    assert samples.shape == (H,) and np.all((samples >= 0) & (samples < 1))
    assert samples[3] > samples[0]                   # sharper heads are sparser
    prof = SparsityProfile(alpha=1.0)
    prof.update_block(0, samples, 0)
    assign, sp = plan_heads_from_profile(prof, 0, grid.size, D, 1)
    cp = HeadParallelDSV(grid, H, D, r, (8, 4, 4), np.clip(sp, 0.0, 0.99), device=cuda,
                         transport="all_to_all")
    out = cp.step(x, wt, q, k, v, do)
    torch.cuda.synchronize()
    assert all(torch.isfinite(t.float()).all() for t in out)


@pytest.mark.parametrize("overlap,fused_out,convert", [("0", "1", "1"), ("1", "0", "1"),
                                                       ("1", "1", "0")])
def test_head_parallel_peer_variants_world1(cuda, pg, monkeypatch, overlap, fused_out, convert):
    # the peer transport's switches — input exchange under the selection / forward
    # (DSV_OVERLAP_IN), outputs stored by the kernels' epilogues (DSV_FUSED_OUT), dK/dV
    # converted in the backward's tail (DSV_BWD_CONVERT) — each turned off against the default
    from paper_2502_07590_b200.cp import HeadParallelDSV

    grid, H, D, r = TokenGrid(8, 16, 16), 4, 128, 16
    sp = np.array([0.5, 0.75, 0.9, 0.95])
    x, wt, q, k, v, do = _inputs(grid, H, D, r, cuda, seed=3)
    base = [t.clone() for t in HeadParallelDSV(grid, H, D, r, (8, 4, 4), sp, device=cuda,
                                               transport="peer").step(x, wt, q, k, v, do)]
    monkeypatch.setenv("DSV_OVERLAP_IN", overlap)
    monkeypatch.setenv("DSV_FUSED_OUT", fused_out)
    monkeypatch.setenv("DSV_BWD_CONVERT", convert)
    cp = HeadParallelDSV(grid, H, D, r, (8, 4, 4), sp, device=cuda, transport="peer")
    got = [t.clone() for t in cp.step(x, wt, q, k, v, do)]
    torch.cuda.synchronize()
    assert torch.equal(got[0], base[0]) and torch.equal(got[1], base[1])
    for a, b in zip(got[2:], base[2:]):
        assert _rel(a, b) <= 1e-5                    # dK / dV: fp32 atomic order only
