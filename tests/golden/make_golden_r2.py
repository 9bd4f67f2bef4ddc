"""Golden vectors for the round-2 host-side additions, produced by running the REFERENCE in
the build container (/root/reference exists only there):
    python tests/golden/make_golden_r2.py
Writes tests/golden/r2_host.npz: synthetic.smooth_qk / smooth_latents draws, the DTSR tensor
bytes of serialize.tensor_bytes, cpmodel.choose_placement / inter_node_traffic decisions,
cpsim.verify_equivalence reports and MessageLog totals on a fixed ledger.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    from dynsparse import cpmodel as CM
    from dynsparse import cpsim as CS
    from dynsparse import grid as GR
    from dynsparse import serialize as SE
    from dynsparse import synthetic as SY

    g = {}
    grid = GR.TokenGrid(4, 6, 8)
    q, k = SY.smooth_qk(grid, 16, np.random.default_rng(3))
    g["smooth_q"], g["smooth_k"] = q, k
    g["smooth_lat"] = SY.smooth_latents(grid, 3, 2, np.random.default_rng(5))
    for i, arr in enumerate([np.arange(12, dtype=np.float64).reshape(3, 4),
                             np.random.default_rng(1).standard_normal((2, 3, 4)).astype(np.float32),
                             np.arange(7, dtype=np.int32), np.arange(6, dtype=np.int64).reshape(2, 3)]):
        g[f"tensor_{i}"] = arr
        g[f"tensor_bytes_{i}"] = np.frombuffer(SE.tensor_bytes(arr), dtype=np.uint8)
    # placement decisions over a few hybrid configs and skewed alphas
    rng = np.random.default_rng(7)
    dec, cross = [], []
    for n, per_node, g_h, g_s in [(4, 2, 2, 2), (8, 4, 2, 4), (8, 4, 4, 2), (8, 2, 2, 4)]:
        cluster = CM.ClusterSpec(n_devices=n, devices_per_node=per_node, intra_bw=1e9,
                                 inter_bw=1e8, compute_rate=1e9, memory_cap=1e12, elem_width=2)
        loads = CM.head_loads(rng.uniform(0.5, 0.95, 8), 4096, 64)
        plan = CM.balance_heads(loads, g_h)
        vals = rng.uniform(0.0, 0.6, (n, n))
        np.fill_diagonal(vals, 0.0)
        alpha = CM.AlphaMatrix(values=vals)
        conf = CM.CPConfig(g_h=g_h, g_s=g_s, placement="hcp-first", plan=plan, objective=0.0,
                           per_device_comp=[], per_device_comm=[], per_device_mem=[])
        dec.append(CM.choose_placement(conf, cluster, alpha, 4096, 64))
        span_alpha = CM.AlphaMatrix(values=vals[:g_s, :g_s] * (1 - np.eye(g_s)))
        for pl in CM.PLACEMENTS:
            cross.append(CM.inter_node_traffic(g_h, g_s, pl, cluster, plan.head_counts(g_h),
                                               span_alpha, 4096, 64))
        g[f"plc_loads_{len(dec) - 1}"] = loads
        g[f"plc_alpha_{len(dec) - 1}"] = vals
        g[f"plc_cfg_{len(dec) - 1}"] = np.array([n, per_node, g_h, g_s])
    g["plc_decisions"] = np.array(dec)
    g["plc_cross"] = np.array(cross, dtype=np.float64)
    # verify_equivalence + MessageLog
    x = rng.standard_normal((2, 8, 4))
    y = x.copy()
    y[1, 3, 2] += 1e-3
    g["veq_x"], g["veq_y"] = x, y
    g["veq_report"] = np.frombuffer(json.dumps(CS.verify_equivalence(y, x, tol=1e-6),
                                               sort_keys=True).encode(), dtype=np.uint8)
    log = CS.MessageLog()
    for i, ph in enumerate(CS.PHASES * 3):
        log.add(ph, i % 4, (i + 1) % 4, 100 * (i + 1))
    g["log_json"] = np.frombuffer(json.dumps(log.to_json(), sort_keys=True).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "r2_host.npz", **g)
    print("wrote", OUT / "r2_host.npz")


if __name__ == "__main__":
    main()
