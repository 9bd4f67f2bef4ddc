"""CPU tier for the round-2 host-side pieces, against goldens written by running the reference
(tests/golden/make_golden_r2.py): synthetic inputs, the DTSR tensor format, placement
choice, cpsim's ledger / equivalence report, the tile tables of ladder voxels, the
reference-name re-exports and the conformance shim."""

import json
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_2502_07590_b200 import cpmodel as CM
from paper_2502_07590_b200 import cpsim as CS
from paper_2502_07590_b200 import serialize as SE
from paper_2502_07590_b200 import synthetic as SY
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.grouping import build_groups, group_tables


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN / "r2_host.npz")


def test_synthetic_draws_equal_reference(gold):
    grid = TokenGrid(4, 6, 8)
    q, k = SY.smooth_qk(grid, 16, np.random.default_rng(3))
    np.testing.assert_array_equal(q, gold["smooth_q"])
    np.testing.assert_array_equal(k, gold["smooth_k"])
    np.testing.assert_array_equal(SY.smooth_latents(grid, 3, 2, np.random.default_rng(5)),
                                  gold["smooth_lat"])


@pytest.mark.parametrize("i", range(4))
def test_tensor_bytes_equal_reference(gold, i, tmp_path):
    arr = gold[f"tensor_{i}"]
    raw = SE.tensor_bytes(arr)
    np.testing.assert_array_equal(np.frombuffer(raw, dtype=np.uint8), gold[f"tensor_bytes_{i}"])
    back = SE.tensor_from_bytes(raw)
    assert back.dtype == arr.dtype and np.array_equal(back, arr)
    SE.save_tensor(tmp_path / "t.bin", arr)
    assert np.array_equal(SE.load_tensor(tmp_path / "t.bin"), arr)
    with pytest.raises(ValueError):
        SE.tensor_from_bytes(b"XXXX" + raw[4:])


def test_choose_placement_and_traffic_equal_reference(gold):
    cross = []
    for c in range(len(gold["plc_decisions"])):
        n, per_node, g_h, g_s = (int(x) for x in gold[f"plc_cfg_{c}"])
        cluster = CM.ClusterSpec(n_devices=n, devices_per_node=per_node, intra_bw=1e9,
                                 inter_bw=1e8, compute_rate=1e9, memory_cap=1e12, elem_width=2)
        plan = CM.balance_heads(gold[f"plc_loads_{c}"], g_h)
        vals = gold[f"plc_alpha_{c}"]
        conf = CM.CPConfig(g_h=g_h, g_s=g_s, placement="hcp-first", plan=plan, objective=0.0,
                           per_device_comp=[], per_device_comm=[], per_device_mem=[])
        assert CM.choose_placement(conf, cluster, CM.AlphaMatrix(values=vals), 4096, 64) == \
            str(gold["plc_decisions"][c])
        span_alpha = CM.AlphaMatrix(values=vals[:g_s, :g_s] * (1 - np.eye(g_s)))
        for pl in CM.PLACEMENTS:
            cross.append(CM.inter_node_traffic(g_h, g_s, pl, cluster, plan.head_counts(g_h),
                                               span_alpha, 4096, 64))
    np.testing.assert_array_equal(np.array(cross), gold["plc_cross"])


def test_cpsim_ledger_and_report_equal_reference(gold):
    log = CS.MessageLog()
    for i, ph in enumerate(CS.PHASES * 3):
        log.add(ph, i % 4, (i + 1) % 4, 100 * (i + 1))
    assert json.dumps(log.to_json(), sort_keys=True).encode() == gold["log_json"].tobytes()
    rep = CS.verify_equivalence(gold["veq_y"], gold["veq_x"], tol=1e-6)
    assert json.dumps(rep, sort_keys=True).encode() == gold["veq_report"].tobytes()
    with pytest.raises(ValueError):
        log.add("no-such-phase", 0, 1, 1)
    assert CS.verify_equivalence(np.zeros((2, 2)), np.zeros((3, 2)))["reason"] == "shape mismatch"


@pytest.mark.parametrize("dims,voxel", [((16, 16, 16), (8, 8, 4)), ((16, 16, 16), (8, 8, 8)),
                                        ((12, 12, 10), (8, 8, 4)), ((16, 40, 50), (8, 4, 4))])
def test_ladder_tile_tables(dims, voxel):
    plan = build_groups(TokenGrid(*dims), voxel)
    rows, size, tg = group_tables(plan.members, split=True)
    if plan.max_group <= 128:
        assert tg is None and rows.shape[0] == plan.n_groups
    else:
        assert tg is not None and rows.shape[0] == tg.size
    parent = np.arange(plan.n_groups) if tg is None else tg
    # every member appears in exactly one tile of its own group, tiles hold 1..128 queries
    seen = np.zeros(plan.grid.size, dtype=np.int64)
    for t in range(rows.shape[0]):
        assert 1 <= size[t] <= 128
        m = rows[t, : size[t]]
        assert set(m.tolist()) <= set(plan.members[parent[t]].tolist())
        assert np.all(rows[t, size[t]:] == m[-1])
        seen[m] += 1
    assert np.all(seen == 1)
    with pytest.raises(ValueError):
        if plan.max_group > 128:
            group_tables(plan.members)          # unsplit tables refuse groups over 128
        else:
            raise ValueError("nothing to refuse")


def test_reference_top_level_names():
    import paper_2502_07590_b200 as ds

    for name in ("CriticalIndexSet", "analyze_distribution", "attention_scores",
                 "critical_kv_oracle", "full_attention", "head_sparsity", "sparse_attention",
                 "TokenGrid", "SampleConfig", "SparsityProfile", "ema_update",
                 "measure_block_sparsity", "sample_queries", "AllocationMeter", "TopKResult",
                 "k_from_sparsity", "streaming_topk", "twopass_select"):
        assert hasattr(ds, name) and name in ds.__all__


def test_conformance_shim_maps_reference_modules():
    sys.path.insert(0, str(ROOT / "conformance" / "shim"))
    try:
        import dynsparse
        from dynsparse.cpsim import run_hybrid_sparse_cp
        from dynsparse.selection import streaming_topk

        import paper_2502_07590_b200.cpsim as cps
        import paper_2502_07590_b200.selection as sel
        assert streaming_topk is sel.streaming_topk and run_hybrid_sparse_cp is cps.run_hybrid_sparse_cp
        assert dynsparse.k_from_sparsity(0.9, 1000) == 100
    finally:
        sys.path.remove(str(ROOT / "conformance" / "shim"))
