"""GPU parity of NEXT-2, the joint global-pose refinement (MIS_F_JOINT_POSE; Eq. 10,
readings A37-A40): the pose is unknown m of the normal equations, with the Eq. 10 priors against
the frame's input pose.  Gates as DESIGN.md §6: the (m+1)-block system within relative 1e-4
(Cauchy-Schwarz scaled), nodes and pose within 0.01 mm / 1e-4 rad of the oracle's MIRROR run."""
import numpy as np
import pytest

import oracle as O
from tests.common import rot, scene_problem, state_f32
from tests.test_gpu_parity import M, check_system, make_ctx, node_state, oracle_params, rot_err

pytestmark = pytest.mark.gpu


def perturbed_pose(P, deg=0.5, dt=(0.8, -0.5, 0.3)):
    """A wrong ORB-SLAM pose (the prior): the frame's pose composed with a small rigid error."""
    R = P[:9].reshape(3, 3)
    return np.concatenate([(R @ rot([1, 2, 3], deg)).ravel(), P[9:] + np.array(dt)])


def joint_ctx(sc, pb, prior, **kw):
    sc = dict(sc)
    sc["pose"] = prior.astype(np.float32)   # the caller's pose is fp32 (mis_set_frame)
    flags = kw.pop("flags", 0) | M.MIS_F_FINAL_ENERGY | M.MIS_F_JOINT_POSE
    return make_ctx(sc, pb, flags=flags, **kw), sc


def ofr(sc):
    return O.Frame(sc["depth"], sc["intr"], np.asarray(sc["pose"], np.float32).astype(np.float64))


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("state", ["identity", "random"])
def test_pose_system_parity(cfg, state):
    sc, pb, fr, _ = scene_problem(cfg)
    prior = perturbed_pose(np.array(fr.s.pose[:]))
    ctx, sc2 = joint_ctx(sc, pb, prior)
    Rt = state_f32(node_state(state, pb.g, seed=21))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    fr2 = ofr(sc2)
    cur = perturbed_pose(np.array(fr2.s.pose[:]), deg=0.2, dt=(-0.3, 0.2, 0.4))   # current != prior: E_r, E_p > 0
    M.mis_dbg_set_pose(ctx.ptr, cur)
    m = pb.g.shape[0]
    gs = M.mis_dbg_system(ctx.ptr, m + 1)
    prm = oracle_params(ctx.params, joint_pose=1, w_r=ctx.params.w_r, w_p=ctx.params.w_p)
    osys = O.system_pose(prm, pb, fr2, Rt, cur)
    assert osys["energy"][4] > 0 and osys["energy"][5] > 0
    o5 = dict(osys)
    o5["energy"] = np.concatenate([osys["energy"][:4], osys["energy"][6:7]])   # GPU energy[4] = weighted total
    check_system(gs, o5, m + 1)
    assert abs(gs["energy"][4] - osys["energy"][6]) <= 1e-4 * osys["energy"][6]
    # the pose row is dense: a block for every node of a kNN tuple or a feature
    assert gs["row_ptr"][m + 1] - gs["row_ptr"][m] > 0.9 * m


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("weights", ["paper", "weak"])
def test_pose_register_parity_mirror(cfg, weights):
    sc, pb, fr, _ = scene_problem(cfg)
    prior = perturbed_pose(np.array(fr.s.pose[:]))
    w = dict(paper={}, weak=dict(w_r=10.0, w_p=1.0))[weights]
    ctx, sc2 = joint_ctx(sc, pb, prior, **w)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert rep["status"] == 0 and rep["solver_cluster"] == 0   # the dense pose row: grid PCG
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    pg = M.mis_get_pose(ctx.ptr)
    fr2 = ofr(sc2)
    prm = oracle_params(ctx.params, joint_pose=1, w_r=ctx.params.w_r, w_p=ctx.params.w_p)
    Ro, po, Eo, nao = O.register_pose(prm, pb, fr2)
    terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
    rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
    assert terr.max() < 0.01, terr.max()
    assert rerr.max() < 1e-4, rerr.max()
    # (the input pose is fp32, so R is orthonormal only to ~1e-7: compare entries, not the arccos of a trace)
    assert np.linalg.norm(pg[9:] - po[9:]) < 0.01 and np.abs(pg[:9] - po[:9]).max() < 1e-4
    moved = np.linalg.norm(po[9:] - np.array(fr2.s.pose[:])[9:])
    assert moved > (0.3 if weights == "weak" else 1e-3), moved    # the pose is refined, not frozen
    assert np.allclose(rep["energy"][:, 4], Eo[:, 6], rtol=1e-3)
    assert np.allclose(rep["energy_pose"][-1], Eo[-1, 4:6], rtol=2e-2, atol=1e-9)
    assert np.abs(rep["n_assoc"] - nao).max() <= max(3, 1e-4 * pb.xyz.shape[0])


def test_pose_warp_and_fuse_use_refined_pose():
    sc, pb, fr, _ = scene_problem("c1")
    prior = perturbed_pose(np.array(fr.s.pose[:]))
    ctx, sc2 = joint_ctx(sc, pb, prior, w_r=10.0, w_p=1.0)
    M.mis_register(ctx.ptr)
    pg = M.mis_get_pose(ctx.ptr)
    n = pb.xyz.shape[0]
    xyz_cam = np.zeros((n, 3), np.float32)
    M.mis_warp(ctx.ptr, xyz_cam)
    mod = M.mis_get_model(ctx.ptr, pb.k)
    exp = mod["xyz"].astype(np.float64) @ pg[:9].reshape(3, 3).T + pg[9:]
    assert np.abs(xyz_cam - exp).max() < 1e-3
    assert np.abs(pg - np.asarray(sc2["pose"], np.float64)).max() > 0.1   # differs from the input pose
    # fusion with the refined pose: the oracle's Alg. 1 / Eq. 12-15 on the same model and that pose
    frp = O.Frame(sc["depth"], sc["intr"], pg)
    o = O.fuse(oracle_params(ctx.params), mod["xyz"], mod["nrm"], mod["rgb"], mod["weight"], mod["stamp"], frp,
               sc["rgb_obs"], 1, M.mis_get_graph(ctx.ptr, np.zeros((pb.g.shape[0], 3), np.float32)))
    n_out, stats = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 1)
    unsure = int((o["key_margin"] <= 1e-6).sum() + (o["gate_margin"] <= 1e-6).sum())
    assert abs(int(stats[0]) - int((o["owner"] >= 0).sum())) <= unsure
    assert abs(int(stats[1]) - o["n_lift"]) <= unsure and stats[0] > 0.5 * n


def test_pose_errors():
    sc, pb, fr, _ = scene_problem("c1")
    with pytest.raises(M.MisError):
        M.Context(M.mis_default_params(flags=M.MIS_F_JOINT_POSE | M.MIS_F_AFFINE))
    with pytest.raises(M.MisError):
        M.Context(M.mis_default_params(k=8, flags=M.MIS_F_JOINT_POSE))
    with pytest.raises(M.MisError):
        M.Context(M.mis_default_params(w_r=-1.0))


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_pose_register_full(cfg):
    """NEXT-2 at the bench configurations (C3: 300k points, 999 nodes, 5 GN x 10 PCG; C4: 2M points,
    ~4000 nodes, 5 GN x 10 PCG; ORB features) with the paper's prior weights and a wrong ORB-SLAM pose:
    nodes and pose against the oracle (on every host core: only its summation order changes)."""
    import os
    from tests.test_gpu_fullsize import problem
    O.set_threads(os.cpu_count() or 1)
    try:
        sc, pb, fr, _ = problem(cfg)
        prior = perturbed_pose(np.array(fr.s.pose[:]))
        ctx, sc2 = joint_ctx(sc, pb, prior)
        rep = M.report_dict(M.mis_register(ctx.ptr))
        assert rep["status"] == 0
        m = pb.g.shape[0]
        Rg = M.mis_get_nodes_f64(ctx.ptr, m)
        pg = M.mis_get_pose(ctx.ptr)
        prm = oracle_params(ctx.params, joint_pose=1, w_r=ctx.params.w_r, w_p=ctx.params.w_p)
        Ro, po, Eo, nao = O.register_pose(prm, pb, ofr(sc2))
    finally:
        O.set_threads(1)
    terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
    rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
    assert terr.max() < 0.01 and rerr.max() < 1e-4, (terr.max(), rerr.max())
    assert np.linalg.norm(pg[9:] - po[9:]) < 0.01 and np.abs(pg[:9] - po[:9]).max() < 1e-4
    assert np.allclose(rep["energy"][:, 4], Eo[:, 6], rtol=1e-3)
