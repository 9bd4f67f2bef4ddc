"""PeerExchange job tables (host only): every rank's forward and return jobs, run
through a byte-level emulator of dsv_copy_jobs over fake peer buffers, must leave
each owner holding exactly the rows the all-to-all form delivers (cpsim.py:125-161,
284-299), for balanced, skewed and contiguous head plans."""

import numpy as np
import pytest
import torch

from paper_2502_07590_b200 import cpmodel
from paper_2502_07590_b200.cp import PeerExchange, plan_heads

BASE = 1 << 44          # fake device address of rank r's buffer: (r + 1) * BASE


class Memory:
    """Address -> bytes for host tensors and fake peer buffers."""

    def __init__(self):
        self.regions = []

    def add(self, base, arr):
        self.regions.append((int(base), arr.reshape(-1).view(np.uint8)))

    def _find(self, addr, n):
        for base, a in self.regions:
            if base <= addr and addr + n <= base + a.size:
                return a, addr - base
        raise AssertionError(f"address {addr:#x}+{n} outside every buffer")

    def run(self, jobs):
        for src, dst, ss, ds, rows, rb in np.asarray(jobs):
            assert src % 16 == 0 and dst % 16 == 0 and ss % 16 == 0 and ds % 16 == 0 and rb % 16 == 0
            assert rows * rb // 16 < 2 ** 31
            for r in range(rows):
                a, o = self._find(src + r * ss, rb)
                b, p = self._find(dst + r * ds, rb)
                b[p:p + rb] = a[o:o + rb]


def _torch_np(t):
    return t.view(torch.int16).numpy()


@pytest.mark.parametrize("world,plan,H", [(2, "balanced", 6), (4, "skewed", 6), (3, "contiguous", 6),
                                          (3, "balanced", 6), (4, "balanced", 6),
                                          (8, "balanced", 24), (8, "skewed", 24), (8, "balanced", 6)])
def test_peer_job_tables_deliver_the_all_to_all_layout(world, plan, H):
    # world 8 with H = 24 is the driver's 8-GPU scaling run (3 heads per rank); H = 6 < 8
    # leaves ranks without heads
    D, r = 16, 8
    L = 24 * world
    chunk = L // world
    sp = np.linspace(0.5, 0.95, H) if plan == "skewed" else np.full(H, 0.9)
    assign = plan_heads(sp, L, D, world, balanced=plan != "contiguous")
    g = torch.Generator().manual_seed(0)
    mk = lambda *s: torch.randn(s, generator=g).to(torch.bfloat16)
    q, k, v, do = (mk(H, L, D) for _ in range(4))
    P = mk(L, 2 * H * r)
    ptrs = [(i + 1) * BASE for i in range(world)]
    ex = [PeerExchange(H, L, D, r, assign, plan_only=(i, world, ptrs)) for i in range(world)]
    mem = Memory()
    bufs = [np.zeros(ex[0].total_elems, dtype=np.int16) for _ in range(world)]
    for i in range(world):
        mem.add(ptrs[i], bufs[i])
    # forward: every rank sends its token chunk of all heads
    keep = []
    for i in range(world):
        sl = slice(i * chunk, (i + 1) * chunk)
        loc = [t[:, sl].contiguous() for t in (q, k, v, do)] + [P[sl].contiguous()]
        keep += loc
        for t in loc:
            mem.add(t.data_ptr(), _torch_np(t))
        mem.run(ex[i]._fwd_jobs(*loc))
    for o in range(world):
        hs = ex[o].my_heads
        nh = len(hs)
        reg = lambda name, w: bufs[o][ex[o].off[name]: ex[o].off[name] + nh * L * w].reshape(nh, L, w)
        for name, t in zip(("q", "k", "v", "do"), (q, k, v, do)):
            np.testing.assert_array_equal(reg(name, D), _torch_np(t[hs]))
        lr = P.view(L, 2, H, r)
        np.testing.assert_array_equal(reg("qlr", r), _torch_np(lr[:, 0, hs].permute(1, 0, 2)))
        np.testing.assert_array_equal(reg("klr", r), _torch_np(lr[:, 1, hs].permute(1, 0, 2)))
    # return: every owner sends its heads' full sequences back to the token owners
    outs = [mk(H, L, D) for _ in range(4)]
    for o in range(world):
        hs = ex[o].my_heads
        mine = [t[hs].contiguous() for t in outs]
        keep += mine
        for t in mine:
            mem.add(t.data_ptr(), _torch_np(t))
        mem.run(ex[o]._back_jobs(mine))
    for i in range(world):
        sl = slice(i * chunk, (i + 1) * chunk)
        for name, t in zip(("o", "dq", "dk", "dv"), outs):
            got = bufs[i][ex[i].off[name]: ex[i].off[name] + H * chunk * D].reshape(H, chunk, D)
            np.testing.assert_array_equal(got, _torch_np(t[:, sl]))
    # ledger arithmetic = the all-to-all's (hcp_comm for the Q/K/V/O part)
    for i in range(world):
        ex[i]._account(("hcp_fwd", 3 * D), ("hcp_bwd_in", D), to_heads=True)
        ex[i]._account(("output_redistribute", D), to_heads=False)
    tot = sum(e.ledger.sent["hcp_fwd"] + e.ledger.sent["output_redistribute"] for e in ex)
    assert tot == sum(e.ledger.received["hcp_fwd"] + e.ledger.received["output_redistribute"] for e in ex)
    for e in ex:
        qkv = max(e.ledger.sent["hcp_fwd"], e.ledger.received["hcp_fwd"])
        assert qkv == cpmodel.hcp_comm(H, len(e.my_heads), L, D, world, 2) * 3 / 4
