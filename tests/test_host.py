"""Host-side logic of the package (CPU only): grouping tables, index sets, the k rule,
the CP planner (vs reference golden vectors and brute force), and the API's
argument validation (raised before any device work, matching the reference's
error contract)."""

import itertools
import math

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2502_07590_b200 import cpmodel, selection
from paper_2502_07590_b200.attention import CriticalIndexSet, head_sparsity, sparse_attention
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.grouping import (VoxelGroupPlan, build_groups, group_tables,
                                            overlap_ratio)


def test_k_from_sparsity_matches_reference_table():
    g = np.load(GOLDEN / "selection.npz")
    for (s, n), k in zip(g["kfs_args"], g["kfs_k"]):
        assert selection.k_from_sparsity(s, int(n)) == k
    with pytest.raises(ValueError):
        selection.k_from_sparsity(1.0, 10)
    with pytest.raises(ValueError):
        selection.k_from_sparsity(0.5, 0)


def test_build_groups_matches_reference():
    g = np.load(GOLDEN / "grouping.npz")
    i = 0
    while f"c{i}_grid" in g:
        plan = build_groups(TokenGrid(*(int(x) for x in g[f"c{i}_grid"])), g[f"c{i}_dims"])
        np.testing.assert_array_equal(plan.proxies, g[f"c{i}_proxies"])
        np.testing.assert_array_equal([m.size for m in plan.members], g[f"c{i}_sizes"])
        np.testing.assert_array_equal(np.concatenate(plan.members), g[f"c{i}_members"])
        i += 1


def test_c2_grouping_shape():
    plan = build_groups(TokenGrid(16, 40, 50), (8, 4, 4))
    sizes = sorted(m.size for m in plan.members)
    assert plan.n_groups == 260 and sizes.count(128) == 240 and sizes.count(64) == 20


def test_group_tables_padding():
    plan = build_groups(TokenGrid(5, 4, 4), (2, 2, 2))
    rows, size = group_tables(plan.members)
    for g, m in enumerate(plan.members):
        assert size[g] == m.size
        np.testing.assert_array_equal(rows[g, : m.size], m)
        assert np.all(rows[g, m.size:] == m[-1])
    with pytest.raises(ValueError):
        group_tables([np.arange(129)])


def test_plan_json_roundtrip_and_validation():
    plan = build_groups(TokenGrid(4, 4, 2), (2, 2, 2))
    again = VoxelGroupPlan.from_json(plan.to_json())
    for a, b in zip(again.members, plan.members):
        np.testing.assert_array_equal(a, b)
    with pytest.raises(ValueError):
        build_groups(TokenGrid(4, 4, 4), (0, 2, 2))
    with pytest.raises(ValueError):
        build_groups(TokenGrid(4, 4, 4), (8, 2, 2))


def test_overlap_ratio():
    sets = [np.array([0, 1]), np.array([2, 3]), np.array([4, 5])]
    assert overlap_ratio(sets, 0) == 0.0
    assert overlap_ratio([np.array([1, 2, 3])] * 4, 0) == 1.0


def test_critical_index_set_contract():
    idx = CriticalIndexSet([np.array([1, 4, 7])] * 3)
    assert idx.uniform_k() == 3 and idx.total_pairs() == 9
    with pytest.raises(ValueError):
        CriticalIndexSet([np.array([3, 1])])
    with pytest.raises(ValueError):
        CriticalIndexSet([np.array([1, 1])])
    with pytest.raises(ValueError):
        CriticalIndexSet([np.array([-1, 2])])
    with pytest.raises(ValueError):
        CriticalIndexSet([np.array([1])], theta=0.0)
    assert head_sparsity(CriticalIndexSet([np.array([3])] * 4), 10) == pytest.approx(0.9)


def test_api_validation_before_device():
    rng = np.random.default_rng(0)
    with pytest.raises(ValueError):
        selection.streaming_topk(rng.standard_normal((3, 2)), rng.standard_normal((4, 2)), 5)
    with pytest.raises(ValueError):
        selection.twopass_select(rng.standard_normal((3, 2)), rng.standard_normal((4, 2)), 0)
    with pytest.raises(ValueError):
        selection.streaming_topk(np.array([[np.nan, 0.0]]), np.ones((2, 2)), 1)
    with pytest.raises(ValueError):
        selection.streaming_topk(rng.standard_normal((3, 2)), rng.standard_normal((4, 3)), 1)
    q = rng.standard_normal((2, 3))
    with pytest.raises(ValueError):
        sparse_attention(q, q, q, CriticalIndexSet([np.array([0]), np.array([], dtype=np.int64)]))
    with pytest.raises(ValueError):
        sparse_attention(q, q, q, CriticalIndexSet([np.array([0])]))


def _brute_min_max(loads, n):
    best = math.inf
    for assign in itertools.product(range(n), repeat=len(loads)):
        bins = np.zeros(n)
        np.add.at(bins, np.asarray(assign), loads)
        best = min(best, bins.max())
    return best


def test_balance_heads_matches_reference_and_brute_force():
    g = np.load(GOLDEN / "cp.npz")
    i = 0
    while f"bh{i}_loads" in g:
        loads, n = g[f"bh{i}_loads"], int(g[f"bh{i}_n"])
        plan = cpmodel.balance_heads(loads, n)
        assert plan.comp_hcp == pytest.approx(float(g[f"bh{i}_comp"]), rel=1e-12)
        if len(loads) <= 7 and n <= 3:
            assert plan.comp_hcp == pytest.approx(_brute_min_max(loads, n), rel=1e-12)
        i += 1
    for n in (2, 4, 8):
        plan = cpmodel.balance_heads(cpmodel.head_loads(g["c4_sparsities"], 131072, 128), n)
        assert plan.comp_hcp == pytest.approx(float(g[f"c4_n{n}_comp"]), rel=1e-9)


def test_rebalance_beats_contiguous_on_skewed_heads():
    g = np.load(GOLDEN / "cp.npz")
    loads = cpmodel.head_loads(g["c4_sparsities"], 131072, 128)
    for n in (2, 4, 8):
        bal = cpmodel.balance_heads(loads, n).comp_hcp
        contiguous = max(loads[i * (24 // n):(i + 1) * (24 // n)].sum() for i in range(n))
        assert bal <= contiguous + 1e-6


def test_hcp_comm_closed_form():
    g = np.load(GOLDEN / "cp.npz")
    for h_total, h_i, s, d, n, w, expect in g["hcp_comm"]:
        assert cpmodel.hcp_comm(int(h_total), int(h_i), int(s), int(d), int(n), int(w)) == expect


def test_solve_hybrid_dominant_head_forces_scp():
    # one dominant head: pure SCP wins (reference tests/test_cpmodel.py:171-183 scenario)
    cluster = cpmodel.ClusterSpec(4, 4, 1e11, 1e10, 1e12, 1e12, 2)
    loads = np.array([100.0, 1.0, 1.0, 1.0]) * 1e9
    alpha = cpmodel.AlphaMatrix(np.full((4, 4), 0.1) - np.eye(4) * 0.1)
    conf = cpmodel.solve_hybrid(loads, alpha, cluster, 4096, 128)
    assert conf.g_s == 4 and conf.g_h == 1
    with pytest.raises(cpmodel.InfeasiblePlanError):
        cpmodel.solve_hybrid(loads, alpha, cpmodel.ClusterSpec(4, 4, 1e11, 1e10, 1e12, 1.0, 2), 4096, 128)
