"""Golden vectors for hybrid head x selective-sequence CP (g_h = 2, g_s = 2, N = 4),
produced by running the REFERENCE simulator `cpsim.run_hybrid_sparse_cp`.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden_hybrid.py
Writes tests/golden/cp_hybrid.npz: inputs, per-query index sets (CSR), the head plan,
the assembled output and every rank's sent / received bytes per ledger phase, for the
hcp-first and scp-first placements.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
PHASES = ("hcp_fwd", "scp_index_exchange", "scp_kv", "output_redistribute")


def main():
    sys.path.insert(0, str(REF))
    from dynsparse import attention as A
    from dynsparse import cpmodel as CM
    from dynsparse import cpsim as CS

    rng = np.random.default_rng(77)
    h, s, d, n = 4, 64, 8, 4
    q = 2.5 * rng.standard_normal((h, s, d))   # peaked softmax: small, uneven critical sets
    k = rng.standard_normal((h, s, d))
    v = rng.standard_normal((h, s, d))
    sets = []
    for hh in range(h):
        scores = A.attention_scores(q[hh], k[hh])
        sets.append(A.critical_kv_oracle(scores, 0.6).indices)
    sparsities = [1.0 - np.mean([x.size for x in per]) / s for per in sets]
    cluster = CM.ClusterSpec(n_devices=n, devices_per_node=n, intra_bw=1e9, inter_bw=1e8,
                             compute_rate=1e9, memory_cap=1e12, elem_width=2)
    plan = CM.balance_heads(CM.head_loads(sparsities, s, d), 2)
    g = {"q": q, "k": k, "v": v, "assign": plan.assignment}
    for placement in ("hcp-first", "scp-first"):
        conf = CM.CPConfig(g_h=2, g_s=2, placement=placement, plan=plan, objective=0.0,
                           per_device_comp=[], per_device_comm=[], per_device_mem=[])
        devs = CS.make_devices(q, k, v, cluster, conf)
        out, log = CS.run_hybrid_sparse_cp(devs, conf, cluster, sets)
        tag = placement.replace("-", "_")
        g[f"{tag}_out"] = out
        for ph in PHASES:
            g[f"{tag}_sent_{ph}"] = np.array([log.sent_by(r, ph) for r in range(n)])
            g[f"{tag}_recv_{ph}"] = np.array([log.received_by(r, ph) for r in range(n)])
    ptr = [0]
    cols = []
    for per in sets:
        for x_ in per:
            cols.append(np.asarray(x_))
            ptr.append(ptr[-1] + len(x_))
    g["ptr"], g["cols"] = np.array(ptr), np.concatenate(cols)
    np.savez_compressed(OUT / "cp_hybrid.npz", **g)
    print("wrote", OUT / "cp_hybrid.npz")


if __name__ == "__main__":
    main()
