"""Oracle: one DSV layer pass on the CPU (test infrastructure / CPU baseline only).

Restates the per-head reference chain on a bounded sample of the workload:
  project (predictor.py:94-100, both sides) -> proxy scores (selection.py:149) ->
  exact top-k (selection.py:178-242) -> grouped sparse attention forward and its
  backward (grouping.py:196-216, trainer.py:110-117), in the reference's float32
  throughput mode (validate.py:16-19 keeps float32).
bench.py times it for `cpu_baseline` and `--impl reference`; the result is
extrapolated from the sampled (head, group) units to the whole layer.
"""

from __future__ import annotations

import time

import numpy as np

from .attention import grouped_attention_bwd, grouped_attention_fwd
from .grouping import build_groups
from .selection import k_from_sparsity, topk_from_scores


class LayerSample:
    def __init__(self, grid_dims, heads, head_dim, d_lr, voxel, sparsity, seed=0):
        self.H, self.D, self.r = heads, head_dim, d_lr
        self.members, self.proxies = build_groups(grid_dims, voxel)
        self.L = int(np.prod(grid_dims))
        self.k = k_from_sparsity(sparsity, self.L)
        rng = np.random.default_rng(seed)
        d_model = heads * head_dim
        self.x = rng.standard_normal((self.L, d_model), dtype=np.float32)
        self.w = (rng.standard_normal((d_model, 2 * d_lr), dtype=np.float32) / np.sqrt(d_model))
        self.q, self.kk, self.v, self.do = (rng.standard_normal((self.L, head_dim), dtype=np.float32)
                                            for _ in range(4))

    @property
    def n_groups(self) -> int:
        return len(self.members)

    def run(self, groups) -> dict:
        """Time one head's projection and the listed groups' select/fwd/bwd."""
        t0 = time.perf_counter()
        lr = self.x @ self.w                                  # [L, 2r] for this head
        t1 = time.perf_counter()
        q_lr, k_lr = lr[:, : self.r], lr[:, self.r:]
        scores = q_lr[self.proxies[groups]] @ k_lr.T          # [g, L] fp32
        idx, _ = topk_from_scores(scores, self.k)
        t2 = time.perf_counter()
        mem = [self.members[g] for g in groups]
        sets = [idx[i] for i in range(len(groups))]
        grouped_attention_fwd(self.q, self.kk, self.v, mem, sets)
        t3 = time.perf_counter()
        grouped_attention_bwd(self.q, self.kk, self.v, mem, sets, self.do)
        t4 = time.perf_counter()
        return {"project": t1 - t0, "select": t2 - t1, "fwd": t3 - t2, "bwd": t4 - t3,
                "groups": len(groups)}

    def layer_seconds(self, timing: dict) -> float:
        """Extrapolate a sample to the full layer (all heads, all groups)."""
        per_group = (timing["select"] + timing["fwd"] + timing["bwd"]) / timing["groups"]
        return self.H * (timing["project"] + per_group * self.n_groups)
