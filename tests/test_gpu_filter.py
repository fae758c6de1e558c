"""GPU parity of NEXT-1, Alg. 3 filtering (`mis_filter`, K14) against oracle O7.

The oracle runs on the GPU model as it stands before the filter (internal order, read back through
mis_get_model: the exact floats the kernels bin), so box decisions are taken on identical fp32
inputs (reading A30) and the two outputs share one order (ascending box key, A33): ids, stamps,
box / survivor / stable counts bit-exact; weights (integer sums) exact; positions, normals and
colours within fp32 accumulation error.  P:244-262.
"""
import numpy as np
import pytest

import oracle as O
from tests.common import scene_problem
from tests.test_gpu_parity import make_ctx

M = pytest.importorskip("paper_1803_02009_b200.mis")
pytestmark = pytest.mark.gpu


def _spacing(xyz):
    ext = xyz.max(0) - xyz.min(0)
    return float(np.sqrt(ext[0] * ext[1] / len(xyz)))


def _oracle_on(mod, grid, frame, tau_time, tau_weight, omega_max):
    return O.filter_points(mod["xyz"], mod["nrm"], mod["rgb"], mod["weight"], mod["stamp"], mod["ids"], grid, frame,
                           tau_time, tau_weight, omega_max)


def _compare(gm, o, stats, n0):
    ns = len(o["weight"])
    assert len(gm["weight"]) == ns
    assert stats[0] == o["cells"] and stats[1] == n0 - ns and stats[3] == ns
    assert stats[2] == int(o["stable"].sum())
    np.testing.assert_array_equal(gm["ids"], o["ids"])
    np.testing.assert_array_equal(gm["stamp"], o["stamp"])
    np.testing.assert_array_equal(gm["weight"].astype(np.float64), o["weight"])
    assert np.abs(gm["xyz"] - o["xyz"]).max() < 1e-3          # mm, fp32 sums of <= ~10 terms at |x| <= 1e3
    assert np.abs(gm["nrm"] - o["nrm"]).max() < 1e-5
    assert np.abs(gm["rgb"] - o["rgb"]).max() < 1e-5


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("box", [0.4, 1.7, 6.0])
def test_filter_parity(cfg, box):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb)
    before = M.mis_get_model(ctx.ptr, pb.k)
    n0 = len(before["weight"])
    grid = box * _spacing(before["xyz"])
    frame, tau_time, tau_weight = 8, 5, 8.0   # synth stamps are in [-5, 0]: every box is stale, light ones go
    n, stats = M.mis_filter(ctx.ptr, grid, frame, tau_time, tau_weight)
    o = _oracle_on(before, grid, frame, tau_time, tau_weight, ctx.params.omega_max)
    assert n == len(o["weight"])
    if box > 1:
        assert 0 < n < n0 and stats[0] < n0   # boxes merge and some are deleted
    gm = M.mis_get_model(ctx.ptr, pb.k)
    _compare(gm, o, stats, n0)
    # A34: the survivors are re-skinned by Eq. 2 against the current nodes
    oi, ow, om = O.skin(gm["xyz"], pb.g, pb.k)
    order = np.argsort(oi, axis=1)
    oi, ow = np.take_along_axis(oi, order, 1), np.take_along_axis(ow, order, 1)
    keep = om > 1e-5
    assert keep.mean() > 0.95
    assert (gm["knn_idx"][keep] == oi[keep]).all()
    assert np.abs(gm["knn_w"][keep] - ow[keep]).max() < 2e-5


def test_filter_keeps_fresh_and_deletes_all_stale():
    """fresh points are retained; with tau_weight above every possible weight and all stamps stale,
    everything goes (empty model), and a later filter on the empty model is a no-op."""
    sc, pb, fr, _ = scene_problem("c1")
    ctx = make_ctx(sc, pb)
    n0 = pb.xyz.shape[0]
    n, stats = M.mis_filter(ctx.ptr, 1e-3, 0, 10, 3.0)   # frame 0: every stamp >= -10, nothing deleted
    assert n == n0 and stats[1] == 0 and stats[0] == n0
    n, stats = M.mis_filter(ctx.ptr, 1e-3, 100, 10, 1e9)
    assert n == 0 and stats[1] == n0 and stats[2] == 0
    n, stats = M.mis_filter(ctx.ptr, 1.0, 100, 10, 1e9)
    assert n == 0 and stats[0] == 0


def test_filter_bad_box_leaves_model_unchanged():
    """Box coordinates outside (-2^30, 2^30): MIS_E_ARG and the model is untouched."""
    sc, pb, fr, _ = scene_problem("c1")
    ctx = make_ctx(sc, pb)
    before = M.mis_get_model(ctx.ptr, pb.k)
    with pytest.raises(M.MisError):
        M.mis_filter(ctx.ptr, 1e-6, 8, 5, 8.0)
    after = M.mis_get_model(ctx.ptr, pb.k)
    for key in ("xyz", "weight", "stamp", "ids", "knn_idx"):
        np.testing.assert_array_equal(after[key], before[key])


def test_fuse_filter_register_chain():
    """Alg. 2 Steps 3-4 then the next frame: fuse, filter (points registered in this frame carry its
    stamp and are never deleted), then a registration on the filtered, re-skinned model."""
    sc, pb, fr, _ = scene_problem("c1")
    ctx = make_ctx(sc, pb)
    rep = M.mis_register(ctx.ptr)
    M.mis_warp(ctx.ptr)
    n1, fst = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 7)
    before = M.mis_get_model(ctx.ptr, pb.k)
    grid = 1.7 * _spacing(before["xyz"])
    n2, stats = M.mis_filter(ctx.ptr, grid, 7, 5, 8.0)
    o = _oracle_on(before, grid, 7, 5, 8.0, ctx.params.omega_max)
    gm = M.mis_get_model(ctx.ptr, pb.k)
    _compare(gm, o, stats, n1)
    assert (gm["stamp"] == 7).sum() >= 1
    fresh_boxes = {tuple(k) for k in np.floor(before["xyz"][before["stamp"] == 7] / np.float32(grid)).astype(int)}
    kept_boxes = {tuple(k) for k in np.floor(gm["xyz"] / np.float32(grid)).astype(int)}
    assert fresh_boxes <= kept_boxes
    rep2 = M.mis_register(ctx.ptr)
    assert rep2.status == 0 and np.isfinite(rep2.energy[0][4])


def test_filter_fullsize_c3():
    """BASELINE's C3 workload in bench.py's launch configuration: model after a full step (register, warp,
    fuse of the 640x480 frame), box = the point spacing, frame 1; every output compared with the oracle."""
    import torch
    from paper_1803_02009_b200 import synth

    sc = synth.make_scene("c3", 1)
    cfg = sc["cfg"]
    n = sc["xyz"].shape[0]
    prm = M.mis_default_params(k=cfg.k, n_nbr=cfg.n_nbr, gn_iters=cfg.gn_iters, pcg_iters=cfg.pcg_iters)
    ctx = M.Context(prm, stream=torch.cuda.current_stream().cuda_stream)
    M.mis_set_model(ctx.ptr, sc["xyz"], sc["nrm"], sc["rgb"], sc["weight"], sc["stamp"], capacity=n + cfg.H * cfg.W + 16)
    M.mis_set_graph(ctx.ptr, sc["g"], sc["nbr"])
    it = sc["intr"]
    M.mis_register(ctx.ptr, sc["depth"], M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"]),
                   sc["pose"], sc["feat_src"], sc["feat_dst"])
    M.mis_warp(ctx.ptr)
    n1, _ = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 1)
    before = M.mis_get_model(ctx.ptr, cfg.k)
    ext = sc["xyz"].max(0) - sc["xyz"].min(0)
    box = float(np.sqrt(ext[0] * ext[1] / n))
    n2, stats = M.mis_filter(ctx.ptr, box, 1, 10, 3.0)
    o = _oracle_on(before, box, 1, 10, 3.0, prm.omega_max)
    assert n2 < n1
    _compare(M.mis_get_model(ctx.ptr, cfg.k), o, stats, n1)
