"""Oracle parity on the headline configuration's own code path (BASELINE.json configs[1], c2).

c2: L = 32000 (16 x 40 x 50), 24 heads, d = 128, r = 16, s = 0.9 (k = 3200), voxel (8, 4, 4)
-> G = 260 groups (240 of 128 queries + 20 remainder groups of 64), 6240 (head, group)
tiles on 148 persistent CTAs (~42 tiles per CTA). This is exactly what bench.py times:
`DSVAttentionLayer.select` (fused K1b+K2), `.forward` (K3f), `.backward` (K3b). Checked:

  * selection: the fused kernel's index lists and thresholds == the oracle's top-k
    (oracle.topk_from_scores, src/selection.py:178-242 rule) on the device's own fp32 proxy
    scores (unfused K1b output), for all 24 x 260 rows — bit-exact;
  * forward O / LSE and backward dQ / dK / dV of three heads (incl. the 20 remainder
    groups) against oracle.grouped_attention_fwd / _bwd (src/grouping.py:196-216,
    src/trainer.py:110-117 autograd) in fp64 on the same bf16 inputs;
  * the persistent multi-tile kernels against one-CTA-per-tile launches
    (DSV_FWD_GRID / DSV_BWD_GRID = tiles, a subprocess): O, LSE and dQ bit-identical,
    dK / dV equal up to fp32 atomic order.

A c4-style case (per-head k 50..95 % sparsity, ragged per-(head, group) counts, 512 tiles on
148 CTAs) covers mixed k in the same persistent path. Measured errors are written to
gpurun_out/parity/*.json (summaries committed under profiles/).

Tolerances (bf16 inputs and outputs, fp32 accumulation, vs fp64), about 2x the errors
measured on a B200 (profiles/r2/parity.md: O rel-L2 2.3e-3, LSE 1.6e-6, gradients 2.4-2.9e-3,
i.e. bf16 output rounding): O max-abs <= 1.5e-2, rel-L2 <= 5e-3; LSE (natural log) max-abs
<= 1e-4; dQ, dK, dV rel-L2 <= 6e-3 (tighter than SURVEY.md 8(c) rule 4's 1e-2 / 2e-2).
"""

import math
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
from conftest import ROOT, parity_report
from paper_2502_07590_b200 import ops
from paper_2502_07590_b200.grid import TokenGrid
from paper_2502_07590_b200.layer import DSVAttentionLayer

pytestmark = pytest.mark.gpu

C2 = {"grid": (16, 40, 50), "H": 24, "D": 128, "r": 16, "voxel": (8, 4, 4), "s": 0.9}
CHECK_HEADS = (0, 11, 23)
TOL = {"o_max": 1.5e-2, "o_rel": 5e-3, "lse_max": 1e-4, "grad_rel": 6e-3}


def _rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def run_layer(cfg, seed=1234, heads=CHECK_HEADS, want_scores=True):
    """Build the layer, run select / forward / backward exactly as bench.py's step does.
    Returns host copies of everything the checks need for `heads`."""
    dev = torch.device("cuda", torch.cuda.current_device())
    grid = TokenGrid(*cfg["grid"])
    H, D = cfg["H"], cfg["D"]
    layer = DSVAttentionLayer(grid, H, D, cfg["r"], cfg["voxel"], cfg["s"], dev)
    L = grid.size
    g = torch.Generator(device=dev).manual_seed(seed)

    def rnd(*shape):
        return torch.randn(shape, device=dev, generator=g).to(torch.bfloat16)

    x, q, k, v, do = rnd(L, H * D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D)
    wt = layer.predictor_weights(seed=0)
    sel = layer.select(x, wt)
    res = {"layer": layer, "fused": layer.fused_select()}
    if want_scores:
        sel_u, scores = layer.select(x, wt, return_scores=True)
        res["scores"] = scores.cpu().numpy()
        res["idx_unfused"] = sel_u.idx.cpu().numpy()
        res["thr_unfused"] = sel_u.thresholds.cpu().numpy()
        del scores
    out, lse = layer.forward(q, k, v, sel)
    dq, dk, dv = layer.backward(q, k, v, out, lse, do, sel)
    acc = layer._acc                     # the fp32 dK / dV accumulators behind dk, dv
    torch.cuda.synchronize()
    res["idx"] = sel.idx.cpu().numpy()
    res["thr"] = sel.thresholds.cpu().numpy()
    hs = list(heads)
    res["heads"] = {}
    for h in hs:
        res["heads"][h] = {
            "q": q[h].double().cpu().numpy(), "k": k[h].double().cpu().numpy(),
            "v": v[h].double().cpu().numpy(), "do": do[h].double().cpu().numpy(),
            "out": out[h].float().cpu().numpy(), "lse": lse[h].cpu().numpy(),
            "dq": dq[h].float().cpu().numpy(), "dk": dk[h].float().cpu().numpy(),
            "dv": dv[h].float().cpu().numpy(), "dk32": acc[0, h].cpu().numpy(),
            "dv32": acc[1, h].cpu().numpy(),
        }
    return res


@pytest.fixture(scope="module")
def c2(cuda):
    return run_layer(C2)


def test_c2_tiles_exceed_persistent_ctas(c2):
    layer = c2["layer"]
    sizes = np.array([m.size for m in layer.plan.members])
    assert layer.G == 260 and int((sizes == 128).sum()) == 240 and int((sizes == 64).sum()) == 20
    assert layer.H * layer.G == 6240 > 148 * 40
    assert c2["fused"], "c2 must take the fused selection path (the bench's path)"


def test_c2_selection_bit_exact(c2):
    layer = c2["layer"]
    k = layer.ks[0]
    assert k == 3200
    idx, thr = c2["idx"], c2["thr"]
    # fused (the bench's path) == unfused on the same proxy scores
    np.testing.assert_array_equal(idx[:, :, :k], c2["idx_unfused"][:, :, :k])
    assert np.array_equal(thr, c2["thr_unfused"])
    # == the oracle's top-k rule on those fp32 scores, every (head, group) row
    sc = c2["scores"]
    mism = 0
    for h in range(layer.H):
        ri, rt = oracle.topk_from_scores(sc[h], k)
        mism += int(np.sum(np.any(idx[h, :, :k] != ri, axis=1)))
        assert np.all(thr[h] == rt.astype(np.float32)), f"head {h} thresholds"
    parity_report("c2_selection", {"rows": layer.H * layer.G, "k": k, "mismatched_rows": mism,
                                   "path": "select_fused (K1b+K2)"})
    assert mism == 0


def _attn_errors(layer, hd, idx_h, ks_h):
    sets = [idx_h[g, :ks_h] for g in range(layer.G)]
    members = layer.plan.members
    ref, ref_lse = oracle.grouped_attention_fwd(hd["q"], hd["k"], hd["v"], members, sets)
    rdq, rdk, rdv = oracle.grouped_attention_bwd(hd["q"], hd["k"], hd["v"], members, sets, hd["do"])
    rem = np.concatenate([m for m in members if m.size < 128])
    return {
        "o_max_abs": float(np.max(np.abs(hd["out"] - ref))),
        "o_rel_l2": _rel_l2(hd["out"], ref),
        "o_rem_groups_max_abs": float(np.max(np.abs(hd["out"][rem] - ref[rem]))),
        "lse_max_abs": float(np.max(np.abs(hd["lse"] * math.log(2.0) - ref_lse))),
        "dq_rel_l2": _rel_l2(hd["dq"], rdq), "dq_max_abs": float(np.max(np.abs(hd["dq"] - rdq))),
        "dk_rel_l2": _rel_l2(hd["dk"], rdk), "dv_rel_l2": _rel_l2(hd["dv"], rdv),
        "dk_fp32acc_rel_l2": _rel_l2(hd["dk32"], rdk), "dv_fp32acc_rel_l2": _rel_l2(hd["dv32"], rdv),
        "dk_max_abs": float(np.max(np.abs(hd["dk"] - rdk))),
        "dv_max_abs": float(np.max(np.abs(hd["dv"] - rdv))),
    }


def _assert_tol(e, where):
    assert e["o_max_abs"] <= TOL["o_max"], (where, e)
    assert e["o_rel_l2"] <= TOL["o_rel"], (where, e)
    assert e["lse_max_abs"] <= TOL["lse_max"], (where, e)
    for key in ("dq_rel_l2", "dk_rel_l2", "dv_rel_l2"):
        assert e[key] <= TOL["grad_rel"], (where, key, e)


def test_c2_attention_vs_oracle(c2):
    layer = c2["layer"]
    errs = {}
    for h in CHECK_HEADS:
        errs[f"head{h}"] = _attn_errors(layer, c2["heads"][h], c2["idx"][h], layer.ks[h])
    parity_report("c2_attention", {"config": "c2 (16x40x50, H=24, D=128, k=3200, voxel 8x4x4)",
                                   "tiles": layer.H * layer.G, "ctas": 148, "tol": TOL, **errs})
    for h, e in errs.items():
        _assert_tol(e, h)


_DUMP = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from test_gpu_c2_parity import run_layer, C2
torch.cuda.set_device(0)
r = run_layer(C2, want_scores=False)
d = {{}}
for h, hd in r["heads"].items():
    for key in ("out", "lse", "dq", "dk32", "dv32"):
        d[f"{{key}}_{{h}}"] = hd[key]
d["idx"] = r["idx"]
np.savez({path!r}, **d)
"""


def test_c2_persistent_equals_per_tile(c2, tmp_path):
    path = str(tmp_path / "per_tile.npz")
    env = dict(os.environ, DSV_FWD_GRID="tiles", DSV_BWD_GRID="tiles", DSV_NO_BUILD="1")
    code = _DUMP.format(root=str(ROOT), tests=str(Path(__file__).parent), path=path)
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    pt = np.load(path)
    assert np.array_equal(pt["idx"], c2["idx"])
    rep = {}
    for h in CHECK_HEADS:
        hd = c2["heads"][h]
        for key in ("out", "lse", "dq"):
            assert np.array_equal(hd[key], pt[f"{key}_{h}"]), f"{key} head {h}: persistent != per-tile"
        for key in ("dk32", "dv32"):
            rel = _rel_l2(hd[key], pt[f"{key}_{h}"])
            rep[f"{key}_head{h}_rel_l2"] = rel
            assert rel < 1e-5, (key, h, rel)
    parity_report("c2_persistent_vs_per_tile", {"o_lse_dq": "bit-identical", **rep})


@pytest.mark.parametrize("D", [128, 64])
def test_mixed_k_ragged_counts_multi_tile(cuda, D):
    # c4-style: per-head k from 50..95 % sparsity, ragged per-(head, group) counts, 512 tiles
    grid = TokenGrid(16, 32, 32)
    H = 4
    dev = cuda
    sp = [0.5, 0.75, 0.9, 0.95]
    layer = DSVAttentionLayer(grid, H, D, 16, (8, 4, 4), sp, dev)
    L, G = grid.size, layer.G
    assert H * G == 512
    g = torch.Generator(device=dev).manual_seed(77 + D)

    def rnd(*shape):
        return torch.randn(shape, device=dev, generator=g).to(torch.bfloat16)

    x, q, k, v, do = rnd(L, H * D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D)
    sel = layer.select(x, layer.predictor_weights(seed=5))
    rng = np.random.default_rng(D)
    counts = np.stack([rng.integers(1, kh + 1, size=G) for kh in layer.ks]).astype(np.int32)
    counts[0, :3] = 1
    counts[1, -1] = layer.ks[1]
    khg = torch.from_numpy(counts).to(dev)
    out, lse = ops.sparse_fwd(q, k, v, layer.grp_rows, layer.grp_size, sel.idx, sel.kcount,
                              layer.scale, kcount_hg=khg)
    dq, dk, dv = ops.sparse_bwd(q, k, v, out, do, lse, layer.grp_rows, layer.grp_size, sel.idx,
                                sel.kcount, layer.scale, kcount_hg=khg)
    torch.cuda.synchronize()
    idx = sel.idx.cpu().numpy()
    errs = {}
    for h in range(H):
        sets = [idx[h, gi, : counts[h, gi]] for gi in range(G)]
        qd, kd, vd, dod = (t[h].double().cpu().numpy() for t in (q, k, v, do))
        ref, ref_lse = oracle.grouped_attention_fwd(qd, kd, vd, layer.plan.members, sets)
        rdq, rdk, rdv = oracle.grouped_attention_bwd(qd, kd, vd, layer.plan.members, sets, dod)
        e = {
            "o_max_abs": float(np.max(np.abs(out[h].float().cpu().numpy() - ref))),
            "o_rel_l2": _rel_l2(out[h].float().cpu().numpy(), ref),
            "lse_max_abs": float(np.max(np.abs(lse[h].cpu().numpy() * math.log(2.0) - ref_lse))),
            "dq_rel_l2": _rel_l2(dq[h].float().cpu().numpy(), rdq),
            "dk_rel_l2": _rel_l2(dk[h].cpu().numpy(), rdk),
            "dv_rel_l2": _rel_l2(dv[h].cpu().numpy(), rdv),
        }
        errs[f"head{h}_k{layer.ks[h]}"] = e
    parity_report(f"mixed_k_ragged_D{D}", {"tiles": H * G, "tol": TOL, **errs})
    for name, e in errs.items():
        _assert_tol(e, name)


@pytest.mark.parametrize("grid_dims,voxel", [((16, 16, 16), (8, 8, 4)), ((16, 16, 16), (8, 8, 8)),
                                              ((12, 12, 10), (8, 8, 4))])
def test_ladder_voxels_over_128_members(cuda, grid_dims, voxel):
    # reference SIZE_LADDER shapes above 128 queries (grouping.py:22-32): each group spans
    # several 128-query tiles that share the group's index row (tile_grp), on tcgen05
    grid = TokenGrid(*grid_dims)
    H, D = 2, 128
    layer = DSVAttentionLayer(grid, H, D, 16, voxel, [0.9, 0.75], cuda)
    assert layer.tile_grp is not None and layer.plan.max_group > 128
    L, G = grid.size, layer.G
    g = torch.Generator(device=cuda).manual_seed(5)

    def rnd(*shape):
        return torch.randn(shape, device=cuda, generator=g).to(torch.bfloat16)

    x, q, k, v, do = rnd(L, H * D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D), rnd(H, L, D)
    sel, scores = layer.select(x, layer.predictor_weights(seed=2), return_scores=True)
    out, lse = layer.forward(q, k, v, sel)
    dq, dk, dv = layer.backward(q, k, v, out, lse, do, sel)
    torch.cuda.synchronize()
    idx, sc = sel.idx.cpu().numpy(), scores.cpu().numpy()
    errs = {}
    for h in range(H):
        kh = layer.ks[h]
        ri, _ = oracle.topk_from_scores(sc[h], kh)
        np.testing.assert_array_equal(idx[h, :, :kh], ri)
        hd = {"q": q[h].double().cpu().numpy(), "k": k[h].double().cpu().numpy(),
              "v": v[h].double().cpu().numpy(), "do": do[h].double().cpu().numpy(),
              "out": out[h].float().cpu().numpy(), "lse": lse[h].cpu().numpy(),
              "dq": dq[h].float().cpu().numpy(), "dk": dk[h].float().cpu().numpy(),
              "dv": dv[h].float().cpu().numpy(), "dk32": layer._acc[0, h].cpu().numpy(),
              "dv32": layer._acc[1, h].cpu().numpy()}
        sets = [idx[h, gi, :kh] for gi in range(G)]
        members = layer.plan.members
        ref, ref_lse = oracle.grouped_attention_fwd(hd["q"], hd["k"], hd["v"], members, sets)
        rdq, rdk, rdv = oracle.grouped_attention_bwd(hd["q"], hd["k"], hd["v"], members, sets, hd["do"])
        e = {"o_max_abs": float(np.max(np.abs(hd["out"] - ref))), "o_rel_l2": _rel_l2(hd["out"], ref),
             "lse_max_abs": float(np.max(np.abs(hd["lse"] * math.log(2.0) - ref_lse))),
             "dq_rel_l2": _rel_l2(hd["dq"], rdq), "dk_rel_l2": _rel_l2(hd["dk"], rdk),
             "dv_rel_l2": _rel_l2(hd["dv"], rdv)}
        errs[f"head{h}"] = e
        _assert_tol(e, f"{voxel} head {h}")
    parity_report(f"ladder_{voxel[0]}x{voxel[1]}x{voxel[2]}_{grid_dims[0]}x{grid_dims[1]}x{grid_dims[2]}",
                  {"groups": G, "tiles": int(layer.grp_rows.shape[0]), **errs})
