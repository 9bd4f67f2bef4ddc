"""Voxel query grouping (reference pkg/src/dynsparse/grouping.py).

A voxel group's members share one critical-KV index list, selected by the group's
proxy query; the tensor-core query tile is 128 queries, so a group of the larger
ladder shapes ((8,8,4) = 256, (8,8,8) = 512 members) spans several tiles that read
the same index row. The plan is built on the host (cheap integer work) and uploaded
once as small device tables consumed by the K3 kernels:

    grp_rows int32 [T, 128]  member token ids per tile, padded by repeating the last member
    grp_size int32 [T]       live members per tile
    tile_grp int32 [T]       the group (index row) of each tile (None when T == G)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .grid import TokenGrid

# Candidate voxel shapes, smallest to largest (grouping.py:22-32).
SIZE_LADDER = (
    (1, 1, 1), (2, 2, 1), (2, 2, 2), (4, 2, 2), (4, 4, 2),
    (4, 4, 4), (8, 4, 4), (8, 8, 4), (8, 8, 8),
)

TILE = 128


@dataclass
class VoxelGroupPlan:
    """Tiling partition of the grid plus one proxy per group (grouping.py:35-61)."""

    grid: TokenGrid
    dims: tuple
    members: list
    proxies: np.ndarray
    _device: dict = field(default_factory=dict, repr=False)

    @property
    def n_groups(self) -> int:
        return len(self.members)

    @property
    def max_group(self) -> int:
        return max(m.size for m in self.members)

    def to_json(self) -> dict:
        return {"grid": list(self.grid.dims), "dims": list(self.dims),
                "proxies": self.proxies.tolist()}

    @classmethod
    def from_json(cls, data: dict) -> "VoxelGroupPlan":
        plan = build_groups(TokenGrid(*data["grid"]), tuple(data["dims"]))
        if plan.proxies.tolist() != list(data["proxies"]):
            raise ValueError("stored proxies do not match the deterministic tiling")
        return plan

    def tables(self, device) -> tuple[torch.Tensor, torch.Tensor]:
        """(grp_rows [G, 128], grp_size [G]) int32 on `device` (cached) — one tile per group;
        plans with groups of more than 128 members use tile_tables."""
        rows, size, tg = self.tile_tables(device)
        if tg is not None:
            raise ValueError(f"groups of up to {self.max_group} members span several 128-query "
                             f"tiles: use tile_tables")
        return rows, size

    def tile_tables(self, device, groups=None):
        """(grp_rows [T, 128], grp_size [T], tile_grp [T] | None) int32 on `device` (cached) for
        all groups or the listed subset (tile_grp then indexes the subset)."""
        key = (str(device), None if groups is None else tuple(int(g) for g in groups))
        if key not in self._device:
            mem = self.members if groups is None else [self.members[int(g)] for g in groups]
            rows, size, tg = group_tables(mem, split=True)
            self._device[key] = (torch.from_numpy(rows).to(device), torch.from_numpy(size).to(device),
                                 None if tg is None else torch.from_numpy(tg).to(device))
        return self._device[key]

    def proxies_tensor(self, device) -> torch.Tensor:
        key = "proxies:" + str(device)
        if key not in self._device:
            self._device[key] = torch.from_numpy(self.proxies.astype(np.int32)).to(device)
        return self._device[key]


def build_groups(grid: TokenGrid, dims) -> VoxelGroupPlan:
    """Tile the grid into voxels of shape dims, clipped at boundaries (grouping.py:64-90).

    Enumeration is t-outer, h, w-inner; the proxy of a voxel is the member at
    floor(len / 2) of its clipped extent along every axis.
    """
    gt, gh, gw = (int(d) for d in dims)
    if min(gt, gh, gw) < 1:
        raise ValueError(f"voxel dims must be positive, got {dims}")
    if gt > grid.frames or gh > grid.height or gw > grid.width:
        raise ValueError(f"voxel dims {dims} exceed grid {grid.dims}")
    T, H, W = grid.dims
    members, proxies = [], []
    for t0 in range(0, T, gt):
        ts = np.arange(t0, min(t0 + gt, T))
        for h0 in range(0, H, gh):
            hs = np.arange(h0, min(h0 + gh, H))
            for w0 in range(0, W, gw):
                ws = np.arange(w0, min(w0 + gw, W))
                flat = (ts[:, None, None] * H + hs[None, :, None]) * W + ws[None, None, :]
                members.append(np.sort(flat.reshape(-1)).astype(np.int64))
                proxies.append(int((ts[ts.size // 2] * H + hs[hs.size // 2]) * W + ws[ws.size // 2]))
    return VoxelGroupPlan(grid=grid, dims=(gt, gh, gw), members=members,
                          proxies=np.asarray(proxies, dtype=np.int64))


def group_tables(members, split: bool = False):
    """Pad member lists to the 128-query tile (host-side). split: a group of more than 128
    members becomes consecutive 128-member tiles of its sorted member list, and the result
    gains the tile -> group map (None when every group is one tile)."""
    tiles, parent = [], []
    for g, m in enumerate(members):
        m = np.asarray(m, dtype=np.int64)
        if m.size == 0 or (m.size > TILE and not split):
            raise ValueError(f"group {g} has {m.size} members; tiles hold 1..{TILE}")
        for t0 in range(0, m.size, TILE):
            tiles.append(m[t0:t0 + TILE])
            parent.append(g)
    T = len(tiles)
    rows = np.empty((T, TILE), dtype=np.int32)
    size = np.empty(T, dtype=np.int32)
    for t, m in enumerate(tiles):
        rows[t, : m.size] = m
        rows[t, m.size:] = m[-1]
        size[t] = m.size
    if not split:
        return rows, size
    tg = None if T == len(members) else np.asarray(parent, dtype=np.int32)
    return rows, size, tg


def overlap_ratio(member_sets: list, proxy_pos: int) -> float:
    """Mean over non-proxy members of |I_m & I_proxy| / |I_m| (grouping.py:93-114)."""
    if not 0 <= proxy_pos < len(member_sets):
        raise ValueError("proxy position outside the member list")
    if len(member_sets) == 1:
        return 1.0
    proxy = np.asarray(member_sets[proxy_pos], dtype=np.int64)
    ratios = []
    for pos, m in enumerate(member_sets):
        if pos == proxy_pos:
            continue
        m = np.asarray(m, dtype=np.int64)
        if m.size == 0:
            raise ValueError("member sets must be nonempty")
        ratios.append(np.intersect1d(m, proxy, assume_unique=True).size / m.size)
    return float(np.mean(ratios))


def grouped_sparse_attention(q, k, v, plan: VoxelGroupPlan, group_sets: list, *, flops=None):
    """Sparse attention where each group's members share one index set (grouping.py:196-216).

    bf16 CUDA tensors with head dim 64/128 run the group-tiled tcgen05 kernel
    directly (128-query tiles; a group of the larger ladder shapes spans several tiles that
    share its index row; ragged per-group set sizes); other
    inputs (numpy / fp32) run the fp32 CUDA-core kernel on the expanded per-query
    lists, matching the reference's expansion (grouping.py:209-216).
    """
    from . import _convert as cv
    from . import ops
    from .attention import CriticalIndexSet, sparse_attention

    if len(group_sets) != plan.n_groups:
        raise ValueError(f"need {plan.n_groups} group index sets, got {len(group_sets)}")
    sets = []
    for g, gs in enumerate(group_sets):
        a = np.asarray(gs.cpu() if isinstance(gs, torch.Tensor) else gs, dtype=np.int64)
        if a.size == 0:
            raise ValueError(f"group {g} has an empty index set")
        sets.append(a)
    tc_ok = (cv.is_torch(q) and cv.is_torch(k) and cv.is_torch(v)
             and all(t.dtype == torch.bfloat16 and t.is_cuda and t.dim() == 2 for t in (q, k, v))
             and q.shape[1] in (64, 128) and k.shape[1] == q.shape[1] and v.shape == k.shape
             and q.shape[0] == plan.grid.size)
    if not tc_ok:
        per_query = [None] * plan.grid.size
        for g, members in enumerate(plan.members):
            for m in members:
                per_query[m] = sets[g]
        return sparse_attention(q, k, v, CriticalIndexSet(per_query), flops=flops)
    q = cv.as_matrix("Q", q)
    dev = q.device
    k_max = max(s.size for s in sets)
    idx = np.zeros((1, plan.n_groups, k_max), dtype=np.int32)
    counts = np.zeros((1, plan.n_groups), dtype=np.int32)
    for g, s in enumerate(sets):
        if np.any(np.diff(s) <= 0) or s[0] < 0 or s[-1] >= k.shape[0]:
            raise ValueError(f"group {g}: indices must be sorted, unique and inside K")
        idx[0, g, : s.size] = s
        counts[0, g] = s.size
    rows, size, tg = plan.tile_tables(dev)
    out, _ = ops.sparse_fwd(q.unsqueeze(0).contiguous(), k.unsqueeze(0).contiguous(),
                            v.unsqueeze(0).contiguous(), rows, size, torch.from_numpy(idx).to(dev),
                            torch.tensor([k_max], dtype=torch.int32, device=dev),
                            kcount_hg=torch.from_numpy(counts).to(dev), tile_grp=tg)
    if flops is not None:
        flops.add_pairs(int(sum(s.size * m.size for s, m in zip(sets, plan.members))), q.shape[1])
        flops.add_per_query(q.shape[0])
    return out[0]


def _softmax_rows_device(q, k, rows=None):
    """fp64 post-softmax scores of q[rows] against every key (attention.py:112-115 math,
    dsv_gemm_f64 + dsv_softmax_rows_f64)."""
    from . import _convert as cv
    from . import ops

    qd = cv.to_device(q, torch.float64)
    if rows is not None:
        qd = qd[torch.as_tensor(np.asarray(rows, dtype=np.int64), device=qd.device)]
    kd = cv.to_device(k, torch.float64)
    sc = ops.gemm_f64(qd.contiguous(), kd.t(), div=float(np.sqrt(q.shape[1])))
    return ops.softmax_rows_f64_(sc)


def _member_sets(q, k, members, theta, k_top):
    """Critical sets of one group's member queries (grouping.py:117-126): the exact top-k_top
    (streaming_topk) or the theta-mass prefix of each member's softmax row."""
    from .attention import _critical_device
    from .selection import streaming_topk

    if k_top is not None:
        rows = streaming_topk(q[members], k, k_top).indices
        return [np.asarray(rows[i]) for i in range(len(members))]
    return _critical_device(_softmax_rows_device(q, k, members), theta)


def select_group_critical(q, k, plan: VoxelGroupPlan, theta: float) -> list:
    """Per-group critical sets selected by each group's proxy query (grouping.py:184-193):
    the theta-mass prefix of the proxy's softmax row, on the device."""
    from . import _convert as cv
    from .attention import _check_unit_interval, _critical_device

    theta = _check_unit_interval("theta", theta, open_low=True)
    q = cv.as_matrix("Q", q)
    k = cv.as_matrix("K", k)
    cv.check_same_cols("Q", q, "K", k)
    return _critical_device(_softmax_rows_device(q, k, plan.proxies), theta)


def calibrate_group_size(qs, ks, grid: TokenGrid, theta: float = 0.9, target_ratio: float = 0.8,
                         *, k_top=None, n_sample_groups: int = 32, seed: int = 0,
                         ladder=SIZE_LADDER) -> tuple:
    """Largest ladder voxel whose sampled mean proxy overlap meets target_ratio
    (grouping.py:129-181). Groups are sampled with the same generator calls as the
    reference (so the same groups are scored); member sets come from the device."""
    from . import _convert as cv

    target_ratio = cv.check_unit_interval("target_ratio", target_ratio, open_low=True)
    if not isinstance(qs, (list, tuple)) and np.ndim(qs) == 2:
        qs, ks = [qs], [ks]
    heads = []
    for q, k in zip(qs, ks):
        q, k = cv.as_matrix("Q", q), cv.as_matrix("K", k)
        cv.check_same_cols("Q", q, "K", k)
        if q.shape[0] != grid.size:
            raise ValueError("Q rows must match the grid token count")
        heads.append((q, k))
    best, best_count = (1, 1, 1), 1
    rng = np.random.default_rng(seed)
    for dims in ladder:
        dims = tuple(int(x) for x in dims)
        if dims == (1, 1, 1):
            continue
        if dims[0] > grid.frames or dims[1] > grid.height or dims[2] > grid.width:
            continue
        plan = build_groups(grid, dims)
        eligible = [g for g in range(plan.n_groups) if plan.members[g].size > 1]
        if not eligible:
            continue
        chosen = rng.choice(len(eligible), size=min(n_sample_groups, len(eligible)), replace=False)
        ratios = []
        for gi in np.asarray(chosen):
            g = eligible[gi]
            members = plan.members[g]
            proxy_pos = int(np.searchsorted(members, plan.proxies[g]))
            for q, k in heads:
                ratios.append(overlap_ratio(_member_sets(q, k, members, theta, k_top), proxy_pos))
        count = int(np.prod(dims))
        if np.mean(ratios) >= target_ratio and count > best_count:
            best, best_count = dims, count
    return best
