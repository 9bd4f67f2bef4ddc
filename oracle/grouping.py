"""Oracle: voxel query grouping (test infrastructure only; see oracle/__init__.py).

Restates grouping.py:64-90 `build_groups`: frame-major flattening
(t * H + h) * W + w (grid.py:37-41); voxels enumerated t-outer, h, w-inner,
clipped at the grid boundary; the proxy is the member at floor(len / 2) of the
clipped extent along every axis.
"""

from __future__ import annotations

import numpy as np


def build_groups(grid_dims, voxel):
    """Returns (members: list of sorted int64 arrays, proxies: int64 array)."""
    T, H, W = (int(x) for x in grid_dims)
    gt, gh, gw = (int(x) for x in voxel)
    if min(gt, gh, gw) < 1 or gt > T or gh > H or gw > W:
        raise ValueError(f"bad voxel {voxel} for grid {grid_dims}")
    members, proxies = [], []
    for t0 in range(0, T, gt):
        ts = np.arange(t0, min(t0 + gt, T))
        for h0 in range(0, H, gh):
            hs = np.arange(h0, min(h0 + gh, H))
            for w0 in range(0, W, gw):
                ws = np.arange(w0, min(w0 + gw, W))
                flat = ((ts[:, None, None] * H + hs[None, :, None]) * W + ws[None, None, :])
                members.append(np.sort(flat.ravel()).astype(np.int64))
                proxies.append((ts[len(ts) // 2] * H + hs[len(hs) // 2]) * W + ws[len(ws) // 2])
    return members, np.asarray(proxies, dtype=np.int64)
