#!/usr/bin/env python
"""Benchmark: DSV dynamic-sparsity attention layer, fwd+bwd tokens/s on B200.

Workload (BASELINE.json configs[1], "c2"): one video-DiT attention block,
L = 32000 tokens (16 x 40 x 50 latent grid), 24 heads, d = 128, bf16, 90%
sparsity (k = 3200 per query group), predictor rank r = 16, voxel groups
(8, 4, 4) -> 260 query tiles. One step = the whole hot path on synthetic
inputs: K1a projection, K1b proxy scores, K2 exact top-k, K3 sparse forward and
backward (dQ, dK, dV). With N > 1 (torchrun) the same layer runs head-parallel
(HCP): each rank holds L/N tokens, NCCL all-to-alls reshard to the heads that
the sparsity-aware planner assigned to it and back (strong scaling).

Prints one JSON line (rank 0). `--impl reference` times the reference's own CPU
implementation of the path (the unmodified `dynsparse` package installed into
baseline/_ref) on a bounded sample of the same workload, on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DiT attn fwd+bwd tokens/s (1/2/4/8 B200) & effective TFLOP/s vs roofline"
GRID = (16, 40, 50)
HEADS, HEAD_DIM, D_LR, VOXEL, SPARSITY = 24, 128, 16, (8, 4, 4), 0.9
WORKLOAD = ("c2: one video-DiT attention block, L=32000 (16x40x50 latent), 24 heads, d=128, "
            "r=16 predictor, sparsity 0.9 (k=3200), voxel groups (8,4,4) -> 260 query tiles")
# --workload: c2 is the headline (BASELINE.json configs[1]); c3 / c4 are the >= 128k-token
# configurations the north_star's scaling target is quoted on
WORKLOADS = {
    "c2": {"grid": GRID, "heads": HEADS, "sparsity": SPARSITY, "desc": WORKLOAD},
    "c3": {"grid": (32, 64, 64), "heads": 16, "sparsity": 0.9,
           "desc": ("c3: 3B-scale video-DiT layer, L=131072 (32x64x64), 16 heads, d=128, r=16, "
                    "sparsity 0.9 (k=13108), voxel groups (8,4,4) -> 1024 query tiles")},
    "c4": {"grid": (32, 64, 64), "heads": 24, "sparsity": "sweep",
           "desc": ("c4: L=131072 (32x64x64), 24 heads, d=128, r=16, per-head sparsity "
                    "0.50..0.95 (shuffled, seed 0), sparsity-aware head re-balancing")},
    "c5": {"grid": (32, 128, 128), "heads": 24, "sparsity": 0.9,
           "desc": ("c5: large video-DiT layer, L=524288 (32x128x128), 24 heads, d=128, r=16, "
                    "sparsity 0.9 (k=52429), voxel groups (8,4,4) -> 4096 query tiles")},
}


def _sparsities(wl: dict, heads: int):
    import numpy as np

    if wl["sparsity"] == "sweep":   # s_h = 0.50 + 0.45 h / (H - 1), shuffled
        s = 0.50 + 0.45 * np.arange(heads) / (heads - 1)
        np.random.default_rng(0).shuffle(s)
        return s
    return wl["sparsity"]


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dsv", choices=["dsv", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=float(os.environ.get("DSV_CPU_BUDGET", 12)))
    ap.add_argument("--unbalanced", action="store_true", help="contiguous head split (no rebalance)")
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--graph", dest="graph", action="store_true",
                    default=os.environ.get("DSV_GRAPH", "1") == "1",
                    help="replay CUDA graphs (default; one per timed step on one GPU; DSV_GRAPH=0 or "
                         "--eager issues the kernels one by one)")
    ap.add_argument("--eager", dest="graph", action="store_false")
    ap.add_argument("--scp", type=int, default=1,
                    help="g_s > 1: hybrid CP, N/g_s head groups x g_s selective-sequence groups")
    ap.add_argument("--voxel", default=None,
                    help="voxel group shape t,h,w (default 8,4,4); the ladder's 8,8,4 / 8,8,8 groups "
                         "span several 128-query tiles")
    ap.add_argument("--dense-heads", type=int, default=0,
                    help="the first M heads are dense residual heads (sparsity 0); under --scp "
                         "they run the ring KV pass (ring.py)")
    return ap.parse_args()


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- CPU reference timing
_SAMPLE = {}
REF_DIR = ROOT / "baseline" / "_ref"


class RefLayerSample:
    """The UNMODIFIED reference (`dynsparse` installed into baseline/_ref from
    /root/reference/pkg) on a bounded sample of the c2 layer, in its
    float32 throughput mode (validate.py:16-19 keeps float32):
      project   predictor.project(X, W_q), project(X, W_k)          one head per sample
      select    selection.streaming_topk(Q_lr[proxies], K_lr, k)     the sampled groups
      fwd       attention.sparse_attention(Q[members], K, V, set)    = grouped_sparse_attention's
                                                                     per-group expansion
      bwd       the reference trainer's sparse autograd (trainer.py:110-117: gather, einsum,
                softmax, einsum) run by torch-CPU on the same group; `_Block.attention` itself
                is self-attention over all S rows (S x k x d gathers: 52 GB at c2), so the
                formulation runs on the sampled queries against all keys
    extrapolated to 24 heads x 260 groups. Without baseline/_ref (not installed) the oracle
    port (oracle.pipeline) stands in and the record says kind "port"."""

    def __init__(self):
        import numpy as np

        sys.path.insert(0, str(REF_DIR))
        from dynsparse import attention, grid, grouping, predictor, selection

        self.mod = {"attention": attention, "predictor": predictor, "selection": selection}
        plan = grouping.build_groups(grid.TokenGrid(*GRID), VOXEL)
        self.members, self.proxies = plan.members, plan.proxies
        self.L = int(np.prod(GRID))
        self.k = selection.k_from_sparsity(SPARSITY, self.L)
        rng = np.random.default_rng(0)
        d_model = HEADS * HEAD_DIM
        self.x = rng.standard_normal((self.L, d_model), dtype=np.float32)
        self.wq, self.wk = (rng.standard_normal((d_model, D_LR), dtype=np.float32) / np.float32(np.sqrt(d_model))
                            for _ in range(2))
        self.q, self.kk, self.v, self.do = (rng.standard_normal((self.L, HEAD_DIM), dtype=np.float32)
                                            for _ in range(4))
        self.kind = "reference"

    @property
    def n_groups(self) -> int:
        return len(self.members)

    def run(self, groups) -> dict:
        import numpy as np
        import torch

        A, P, Sel = self.mod["attention"], self.mod["predictor"], self.mod["selection"]
        t0 = time.perf_counter()
        q_lr = P.project(self.x, self.wq)
        k_lr = P.project(self.x, self.wk)
        t1 = time.perf_counter()
        sets = Sel.streaming_topk(q_lr[self.proxies[groups]], k_lr, self.k).indices
        t2 = time.perf_counter()
        for i, g in enumerate(groups):
            mem = self.members[g]
            A.sparse_attention(self.q[mem], self.kk, self.v, A.CriticalIndexSet([sets[i]] * mem.size))
        t3 = time.perf_counter()
        t_bwd = 0.0
        kt = torch.from_numpy(self.kk)[None, None].requires_grad_(True)    # [B, H, S, dk]
        vt = torch.from_numpy(self.v)[None, None].requires_grad_(True)
        for i, g in enumerate(groups):
            mem = self.members[g]
            qt = torch.from_numpy(self.q[mem])[None, None].requires_grad_(True)
            idx = torch.from_numpy(np.asarray(sets[i], dtype=np.int64)).expand(mem.size, -1)
            k_sel = torch.stack([kt[0][:, idx]])
            v_sel = torch.stack([vt[0][:, idx]])
            logits = torch.einsum("bhqd,bhqkd->bhqk", qt, k_sel) / math.sqrt(HEAD_DIM)
            out = torch.einsum("bhqk,bhqkd->bhqd", torch.softmax(logits, dim=-1), v_sel)
            dout = torch.from_numpy(self.do[mem])[None, None]
            tb = time.perf_counter()
            out.backward(dout)
            t_bwd += time.perf_counter() - tb
        return {"project": t1 - t0, "select": t2 - t1, "fwd": t3 - t2, "bwd": t_bwd,
                "groups": len(groups)}

    def layer_seconds(self, timing: dict) -> float:
        per_group = (timing["select"] + timing["fwd"] + timing["bwd"]) / timing["groups"]
        return HEADS * (timing["project"] + per_group * self.n_groups)


def _sample():
    if "s" not in _SAMPLE:
        if (REF_DIR / "dynsparse").is_dir():
            _SAMPLE["s"] = RefLayerSample()
        else:
            from oracle.pipeline import LayerSample

            smp = LayerSample(GRID, HEADS, HEAD_DIM, D_LR, VOXEL, SPARSITY)
            smp.kind = "port"
            _SAMPLE["s"] = smp
    return _SAMPLE["s"]


def cpu_oracle(budget_s: float, warm: bool = True) -> dict:
    """The reference CPU path on a bounded sample of the c2 workload (RefLayerSample)."""
    import numpy as np  # noqa: F401  (RefLayerSample.run)
    import torch

    torch.set_num_threads(_cores())
    smp = _sample()
    if warm:
        smp.run([0])
    tot = {"project": 0.0, "select": 0.0, "fwd": 0.0, "bwd": 0.0, "groups": 0}
    g = 0
    t_start = time.perf_counter()
    n_proj = 0
    while True:
        groups = [(g + i * 67) % smp.n_groups for i in range(4)]
        t = smp.run(groups)
        for key in ("project", "select", "fwd", "bwd"):
            tot[key] += t[key]
        tot["groups"] += t["groups"]
        n_proj += 1
        g += 1
        if time.perf_counter() - t_start >= budget_s:
            break
    tot["project"] /= n_proj
    layer_s = smp.layer_seconds(tot)
    what = ("unmodified reference (baseline/_ref dynsparse: project, streaming_topk, "
            "sparse_attention; trainer autograd formulation for the backward), float32"
            if smp.kind == "reference" else "oracle port (oracle.pipeline), float32")
    return {"tokens_per_s": smp.L / layer_s, "layer_seconds": layer_s, "kind": smp.kind,
            "sample": (f"{tot['groups']} (head, group) query tiles of <= 128 + {n_proj} one-head "
                       f"projections, {what}; extrapolated to 24 heads x 260 groups"),
            "stage_s": {k: tot[k] for k in ("select", "fwd", "bwd")},
            "wall_s": time.perf_counter() - t_start}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(gpu_index), "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------- GPU arm
def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16": d.get("bf16_tflops", 1590.0),
                "bf16_sustained": d.get("bf16_tflops_sustained", 1400.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "source": "fallback"}


def _traffic() -> dict:
    p = ROOT / "profiles" / "traffic.json"
    return json.loads(p.read_text()) if p.exists() else {}


def run_gpu(args) -> None:
    global VOXEL
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2502_07590_b200 import ops
    from paper_2502_07590_b200.grid import TokenGrid
    from paper_2502_07590_b200.grouping import build_groups
    from paper_2502_07590_b200.layer import DSVAttentionLayer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.voxel:
        VOXEL = tuple(int(x) for x in args.voxel.split(","))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = WORKLOADS[args.workload]
    grid = TokenGrid(*wl["grid"])
    L, H, D = grid.size, wl["heads"], HEAD_DIM
    sparsity = _sparsities(wl, H)
    if args.dense_heads:
        import numpy as np

        sparsity = np.broadcast_to(np.asarray(sparsity, dtype=np.float64), (H,)).copy()
        sparsity[:args.dense_heads] = 0.0
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)

    def rnd(*shape):
        return torch.randn(shape, device=dev, generator=gen).to(torch.bfloat16)

    if world == 1:
        layer = DSVAttentionLayer(grid, H, D, D_LR, VOXEL, sparsity, dev)
        wt = layer.predictor_weights(seed=0)
        x, q, k, v, do = rnd(L, H * D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D)
        # "bwd_kernel": the backward kernel alone (the roofline's unit); "convert": the dK/dV
        # fp32 -> bf16 conversion that completes layer.backward
        stage_names = ("select", "fwd", "bwd_kernel", "convert")

        def step(ev=None):
            sel = layer.select(x, wt)
            if ev is not None:
                ev[0].record()
            out, lse = layer.forward(q, k, v, sel)
            if ev is not None:
                ev[1].record()
            res = layer.backward(q, k, v, out, lse, do, sel,         # accumulators zeroed by
                                 kernel_done=ev[2] if ev is not None else None)   # the forward
            if ev is not None:
                ev[3].record()
            return res
        # project, proxy gather, (scores gemm + topk | fused select: main + finish + list-mode
        # re-run launch), fwd (persistent + list-mode re-run), bwd (+ 2x f32->bf16 unless the
        # backward converts in its tail)
        launches_per_step = (8 if layer.fused_select() else 7) + (
            0 if os.environ.get("DSV_BWD_CONVERT", "1") != "0" else 2)
        work = layer.work()
    else:
        from paper_2502_07590_b200.cp import HeadParallelDSV, HybridDSV

        if args.scp > 1 or args.dense_heads:   # dense residual heads: ring KV pass (g_s = 1: local)
            cp = HybridDSV(grid, H, D, D_LR, VOXEL, sparsity, world // args.scp, args.scp,
                           balanced=not args.unbalanced, device=dev)
        else:
            cp = HeadParallelDSV(grid, H, D, D_LR, VOXEL, sparsity, balanced=not args.unbalanced,
                                 device=dev)
        layer = cp.local
        chunk = L // world
        g0 = torch.Generator(device="cpu").manual_seed(0)
        wt = (torch.randn((2 * H * D_LR, H * D), generator=g0) / math.sqrt(H * D)).to(torch.bfloat16).to(dev)
        x, q, k, v, do = rnd(chunk, H * D), rnd(H, chunk, D), rnd(H, chunk, D), rnd(H, chunk, D), rnd(H, chunk, D)
        stage_names = ()

        def step(ev=None):
            return cp.step(x, wt, q, k, v, do)
        launches_per_step = (cp.launches_per_step() if getattr(cp, "transport", None) == "peer"
                             and hasattr(cp, "launches_per_step") else 8 + 8)
        if args.dense_heads:        # ring: per hop attend + merge, grad + 2 accumulations; 2 converts
            launches_per_step += 5 * args.scp + 2
        # the kernel rooflines below are of the sparse kernels (the `fwd` / `bwd` stages);
        # dense residual heads (ring stages) are counted in effective_tflops only
        work = layer.work() if layer is not None else None

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    eager_step = step
    if args.graph and args.dense_heads:
        args.graph = False   # the ring KV pass issues host-sized NCCL P2P hops
    graph_evs = None
    if args.graph:
        # CUDA graphs: the host issues one launch per step instead of ~10-20 kernels. On one
        # GPU every timed step gets its own graph (one shared memory pool, replayed in capture
        # order) whose stage boundaries are external CUDA events — event record nodes on the
        # launching stream — so the per-stage (and the roofline kernel's) times are measured
        # live over the whole timed region, not in extra steps outside it
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        graphs, pool = [], None
        per_step = world == 1 and bool(stage_names)
        graph_evs = [] if per_step else None
        for _ in range(args.steps if per_step else 1):
            g = torch.cuda.CUDAGraph()
            ev = ([torch.cuda.Event(enable_timing=True, external=True)
                   for _ in range(len(stage_names) + 1)] if per_step else None)
            with torch.cuda.graph(g, pool=pool):
                if ev is not None:
                    ev[0].record()
                step(ev[1:] if ev is not None else None)
            pool = g.pool()
            graphs.append(g)
            if per_step:
                graph_evs.append(ev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        replay_i = [0]

        def step(ev=None):
            graphs[replay_i[0] % len(graphs)].replay()
            replay_i[0] += 1
        eager_stage_names, stage_names = stage_names, ()
        for _ in range(len(graphs)):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    clocks = ClockSampler(local_rank)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stage_names))]
           for _ in range(args.steps)]
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_begin = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_begin.record()
    for i in range(args.steps):
        starts[i].record()
        step(evs[i] if stage_names else None)
    t_end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed = t_begin.elapsed_time(t_end)
    if world > 1:
        tt = torch.tensor([elapsed], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    ms = elapsed / args.steps
    stage_ms = {}
    if stage_names:
        for si, name in enumerate(stage_names):
            vals = [(starts[i] if si == 0 else evs[i][si - 1]).elapsed_time(evs[i][si])
                    for i in range(args.steps)]
            stage_ms[name] = sum(vals) / len(vals)
    if graph_evs:
        # per-stage times of the timed replays (each graph's events hold its last replay:
        # exactly one, inside the timed loop); mean over the K steps
        stage_ms = {}
        for si, name in enumerate(eager_stage_names):
            vals = [graph_evs[i][si].elapsed_time(graph_evs[i][si + 1]) for i in range(len(graph_evs))]
            stage_ms[name] = sum(vals) / len(vals)
    if world > 1:
        # extra (untimed) eager steps; per-phase events on the compute stream of the last
        eager_step()
        cp.marks = []
        eager_step()
        stage_ms = cp.phase_ms()
        cp.marks = None

    # ---- e2e through the public layer API with host-resident inputs and outputs
    e2e = None
    if not args.no_e2e:
        from paper_2502_07590_b200.layer import HostPipeline

        host = [t.cpu().pin_memory() for t in (x, q, k, v, do)]
        pipe = HostPipeline(host, dev)
        h2d = pipe.h2d_bytes

        def dev_step(xb, qb, kb, vb, dob):
            if world == 1:
                return layer.step(xb, wt, qb, kb, vb, dob)
            return cp.step(xb, wt, qb, kb, vb, dob)

        for _ in pipe.run(dev_step, [host] * 2, reused=world > 1):
            pass
        pipe.drain()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n_e2e = max(3, args.steps)        # the same K as the device-timed loop
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # every step: pinned H2D of its own inputs (overlapping the previous step) and the D2H
        # of its results O, dQ, dK, dV into pinned host buffers (overlapping the next step);
        # the clock starts before the first copy and stops after the last result landed
        a.record()
        for _ in pipe.run(dev_step, [host] * n_e2e, reused=world > 1):
            pass
        pipe.drain()
        b.record()
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / n_e2e
        if world > 1:
            tt = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        e2e = {"value": L / (e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": pipe.d2h_bytes,
               "api": ("DSVAttentionLayer.step" if world == 1 else "HeadParallelDSV.step")
               + " via HostPipeline (pinned H2D of step i+1 and D2H of step i-1's O, dQ, dK, dV "
                 "overlap step i; full-duplex PCIe)"}

    if args.graph:
        del graphs, step                 # release the captured graphs before the groups go
        torch.cuda.synchronize()
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks = _peaks()
    value = L / (ms / 1e3)
    from paper_2502_07590_b200.selection import k_from_sparsity

    all_ks = [k_from_sparsity(float(s_h), L) for s_h in np.broadcast_to(sparsity, (H,))]
    G_all = len(build_groups(grid, VOXEL).members)
    # whole-layer algorithmic work (all heads), whatever this rank holds
    tot_flops = (2 * L * (H * D) * (2 * D_LR * H) + 2 * H * G_all * L * D_LR
                 + 14 * L * sum(all_ks) * D)
    dense_eq = 4 * L * L * D * H * 3.5
    res = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: N(0,1) X, Q, K, V, dO in bf16; random-init predictor W (N(0,1/sqrt(d)))",
        "config": {"workload": wl["desc"], "tokens": L, "heads": H, "head_dim": D, "d_lr": D_LR,
                   "sparsity": (SPARSITY if args.workload == "c2" else
                                [round(float(x), 4) for x in np.broadcast_to(sparsity, (H,))]),
                   "k_per_group": all_ks[0] if args.workload == "c2" else all_ks,
                   "voxel": list(VOXEL),
                   "groups": layer.G if world == 1 else len(build_groups(grid, VOXEL).members),
                   **({"voxel_override": True, "tiles_per_head": int(layer.grp_rows.shape[0])}
                      if args.voxel else {}),
                   "parallelism": ("single" if world == 1 else f"hcp{world}" if args.scp == 1
                                   else f"hcp{world // args.scp}xscp{args.scp}"),
                   "head_plan": "balance_heads" if not args.unbalanced else "contiguous",
                   **({"dense_heads": args.dense_heads} if args.dense_heads else {}),
                   "l2_note": f"inputs (X, Q, K, V, dO: {5 * L * H * D * 2 / 1e9:.2f} GB) exceed the 126 MB L2"},
        "effective_tflops": {"algorithmic": tot_flops / (ms / 1e3) / 1e12,
                             "dense_equivalent": dense_eq / (ms / 1e3) / 1e12},
        "gpu_launches": launches_per_step * args.steps,
        "cuda_graph": bool(args.graph),
        "clocks": clk,
    }
    if stage_ms:
        res["stage_ms"] = stage_ms
    if stage_ms and "bwd_kernel" in stage_ms:            # one GPU: bwd = kernel + conversion
        stage_ms["bwd"] = stage_ms["bwd_kernel"] + stage_ms.pop("convert")
    if stage_ms and work is not None and "bwd" in stage_ms:
        # dominant kernel: sparse backward (tensor-bound by design; scatter-add to L2 limits it)
        bwd_ms = stage_ms.get("bwd_kernel", stage_ms["bwd"])
        achieved = work["bwd_flops"] / (bwd_ms / 1e3) / 1e12
        traffic = _traffic().get("sparse_bwd_kernel")
        res["roofline"] = {"kernel": "sparse_bwd_kernel<128>", "bound": "tensor",
                           "achieved": achieved, "peak": peaks["bf16_sustained"], "unit": "TFLOP/s",
                           "frac": achieved / peaks["bf16_sustained"],
                           "peak_source": f"{peaks['source']} bf16 sustained",
                           "traffic": traffic, "algorithmic_flops": work["bwd_flops"]}
        fwd_ach = work["fwd_flops"] / (stage_ms["fwd"] / 1e3) / 1e12
        # the L2-side bounds of the attention kernels (measured caps on this B200:
        # random 256 B row gathers ~14 TB/s, tools/gather_bench.cu; fp32 reductions into
        # L2-resident rows ~5.5 TB/s, tools/scatter_bench.cu)
        pair_rows = work["fwd_flops"] / (4 * D)              # sum over (head, query) of k
        gather_b = 2 * (pair_rows / 128) * D * 2             # K and V rows per 128-query tile
        red_b = 2 * (pair_rows / 128) * D * 4                # dK and dV fp32 adds per tile
        res["kernels_roofline"] = {
            "sparse_fwd": {"ms": stage_ms["fwd"], "achieved_tflops": fwd_ach,
                           "frac": fwd_ach / peaks["bf16_sustained"],
                           "l2_gather_tbs": gather_b / (stage_ms["fwd"] / 1e3) / 1e12,
                           "l2_gather_frac_of_14tbs": gather_b / (stage_ms["fwd"] / 1e3) / 14e12},
            "sparse_bwd_l2": {"fp32_reduction_tbs": red_b / (bwd_ms / 1e3) / 1e12,
                              "frac_of_5.5tbs": red_b / (bwd_ms / 1e3) / 5.5e12,
                              "gather_tbs": gather_b / (bwd_ms / 1e3) / 1e12},
            "select(project+scores+topk)": {
                "ms": stage_ms["select"],
                # SURVEY 8(d)'s selection roofline is the unfused K2's: the fp32 score matrix
                # read from HBM plus the index lists written (topk_bytes). The fused path
                # never stores those scores, so this is the bound the design removed, not
                # one it runs against (its own compulsory HBM traffic is ~0.1 GB)
                "unfused_k2_hbm_floor_ms": work["topk_bytes"] / (peaks["hbm_gbs"] * 1e9) * 1e3,
                "frac_of_unfused_k2_floor": (work["topk_bytes"] / (peaks["hbm_gbs"] * 1e9) * 1e3)
                / stage_ms["select"]},
        }
    if e2e is not None:
        res["e2e"] = e2e
    if world == 1 and args.workload == "c2" and os.environ.get("DSV_CPU_BASELINE", "1") != "0":
        cb = cpu_oracle(args.cpu_budget)
        res["cpu_baseline"] = {"value": cb["tokens_per_s"], "unit": "tokens/s", "cores": _cores(),
                               "kind": cb["kind"], "sample": cb["sample"], "same_config": True,
                               "threads_note": "numpy/OpenBLAS default threads = all cores; "
                                               "torch.set_num_threads(cores)"}
    print(json.dumps(res))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    budget = float(os.environ.get("DSV_REF_STEP_BUDGET", 3.0))
    cpu_oracle(0.0)  # warm-up, untimed
    for _ in range(max(args.warmup, 3) - 1):
        cpu_oracle(0.0, warm=False)
    vals, walls = [], []
    for _ in range(args.steps):
        r = cpu_oracle(budget, warm=False)
        vals.append(r["tokens_per_s"])
        walls.append(r["layer_seconds"])
        sample, kind = r["sample"], r["kind"]
    value = statistics.median(vals)
    res = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
           "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
           "ms_per_step": statistics.median(walls) * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic: N(0,1) X, Q, K, V, dO (float32, reference throughput mode)",
           "config": {"workload": WORKLOAD, "tokens": 32000, "heads": HEADS, "head_dim": HEAD_DIM,
                      "sparsity": SPARSITY, "voxel": list(VOXEL)},
           "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": _cores(), "kind": kind,
                            "sample": sample, "same_config": True},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(res))


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
