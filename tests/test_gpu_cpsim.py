"""cpsim's reference API on the device against the REFERENCE simulator's goldens.

tests/golden/cp_hybrid.npz was written by running the reference's own
`cpsim.run_hybrid_sparse_cp` (tests/golden/make_golden_hybrid.py): g_h = 2, g_s = 2, N = 4,
both placements. Here `paper_2502_07590_b200.cpsim` runs the same pipeline with its logical
ranks on the visible GPUs (device-to-device / NVLink peer copies, fp64 CSR attention): the
assembled output must match within 1e-12 and every rank's sent / received bytes per phase
must be identical.
"""

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2502_07590_b200 import cpsim
from paper_2502_07590_b200.cpmodel import CPConfig, ClusterSpec, HcpPlan

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("placement", ["hcp-first", "scp-first"])
def test_run_hybrid_sparse_cp_equals_reference_golden(cuda, placement):
    g = np.load(GOLDEN / "cp_hybrid.npz")
    H, S, D = g["q"].shape
    ptr, cols = g["ptr"], g["cols"]
    sets = [[cols[ptr[h * S + s]:ptr[h * S + s + 1]] for s in range(S)] for h in range(H)]
    cluster = ClusterSpec(n_devices=4, devices_per_node=4, intra_bw=1e9, inter_bw=1e8,
                          compute_rate=1e9, memory_cap=1e12, elem_width=2)
    plan = HcpPlan(assignment=np.asarray(g["assign"]), device_loads=np.zeros(2), comp_hcp=0.0,
                   optimal=True)
    conf = CPConfig(g_h=2, g_s=2, placement=placement, plan=plan, objective=0.0,
                    per_device_comp=[], per_device_comm=[], per_device_mem=[])
    devs = cpsim.make_devices(g["q"], g["k"], g["v"], cluster, conf)
    assert [d.device.index for d in devs] == [r % torch.cuda.device_count() for r in range(4)]
    out, log = cpsim.run_hybrid_sparse_cp(devs, conf, cluster, sets)
    tag = placement.replace("-", "_")
    np.testing.assert_allclose(out, g[f"{tag}_out"], atol=1e-12)
    for ph in cpsim.PHASES:
        np.testing.assert_array_equal([log.sent_by(r, ph) for r in range(4)], g[f"{tag}_sent_{ph}"])
        np.testing.assert_array_equal([log.received_by(r, ph) for r in range(4)], g[f"{tag}_recv_{ph}"])
