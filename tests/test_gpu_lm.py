"""NEXT-3 on the GPU: Levenberg-Marquardt registration (MIS_F_LM, reading
A29) through the C-ABI against the fp64 oracle's LM in MIRROR mode (same G, same P):
identical accept / reject decisions wherever the oracle's trial energy is not within a
relative 1e-5 of the last accepted one, trial energies within 1e-3 relative, converged
nodes within the north_star gates (0.01 mm / 1e-4 rad), and the returned state is the last
accepted one.  The cluster PCG carries the decisions on the device (no host round trip)."""
import numpy as np
import pytest

import oracle as O
from tests.common import scene_problem
from tests.test_gpu_parity import make_ctx, oracle_params, rot_err

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1803_02009_b200.mis")


def _near_ties(E, acc, rel):
    """Iterations whose decision is within `rel` of the last accepted energy (oracle side)."""
    out, e_acc = [], None
    for i, (e, a) in enumerate(zip(E, acc)):
        if i > 0 and abs(e - e_acc) <= rel * abs(e_acc):
            out.append(i)
        if a:
            e_acc = e
    return out


@pytest.mark.parametrize("cfg,G", [("c1", 8), ("c2", 6), ("c3", 5)])
def test_lm_parity_mirror(cfg, G):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb, flags=M.MIS_F_LM, gn_iters=G)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert rep["status"] == 0 and rep["solver_cluster"] > 0
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    prm = oracle_params(ctx.params, lm=1, lm_mu0=1e-3, gn_iters=G)
    Ro, Eo, nao, acco = O.register(prm, pb, fr, with_accepted=True)
    ties = _near_ties(Eo[:, 4], acco, 1e-5)
    acc_g = rep["accepted"].astype(int)
    # decisions (the first near tie ends the comparison: states may legitimately differ after it)
    stop = ties[0] if ties else G + 1
    assert (acc_g[:stop] == acco[:stop]).all(), (acc_g, acco, ties)
    assert np.allclose(rep["energy"][:stop, 4], Eo[:stop, 4], rtol=1e-3)
    if not ties:
        terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
        rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
        assert terr.max() < 0.01, terr.max()
        assert rerr.max() < 1e-4, rerr.max()
    # GPU-side invariants: accepted energies strictly decrease; the returned state is the last accepted
    ea = rep["energy"][acc_g == 1, 4]
    assert (np.diff(ea) < 0).all(), ea
    Ef = O.system(prm, pb, fr, Rg)["energy"][4]
    assert abs(Ef - ea[-1]) <= 1e-3 * ea[-1], (Ef, ea[-1])


def test_lm_rejects_and_restores():
    """A run long enough to reach the noise floor rejects trials (both branches exercised on
    the device) and still matches the oracle's decisions up to the first near tie."""
    sc, pb, fr, _ = scene_problem("c1")
    G = 12
    ctx = make_ctx(sc, pb, flags=M.MIS_F_LM, gn_iters=G)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    acc_g = rep["accepted"].astype(int)
    prm = oracle_params(ctx.params, lm=1, lm_mu0=1e-3, gn_iters=G)
    _, Eo, _, acco = O.register(prm, pb, fr, with_accepted=True)
    assert (acco == 0).any()
    ties = _near_ties(Eo[:, 4], acco, 1e-5)
    stop = ties[0] if ties else G + 1
    assert (acc_g[:stop] == acco[:stop]).all(), (acc_g, acco, ties)
    assert (acc_g == 0).any()


def _check_lm(rep, Eo, acco, G, tot=4):
    ties = _near_ties(Eo[:, tot], acco, 1e-5)
    acc_g = rep["accepted"].astype(int)
    stop = ties[0] if ties else G + 1
    assert (acc_g[:stop] == acco[:stop]).all(), (acc_g, acco, ties)
    assert np.allclose(rep["energy"][:stop, 4], Eo[:stop, tot], rtol=1e-3)
    ea = rep["energy"][acc_g == 1, 4]
    assert (np.diff(ea) < 0).all(), ea
    return ties


@pytest.mark.parametrize("cfg,G", [("c1", 12), ("c2", 6)])
def test_lm_grid_parity_mirror(cfg, G):
    """LM in the pipelined grid PCG (MIS_F_GRID_SOLVER: the C4 / C5 solver): the same decisions,
    energies and nodes as the oracle's LM (both branches exercised at C1, G = 12)."""
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb, flags=M.MIS_F_LM | M.MIS_F_GRID_SOLVER, gn_iters=G)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert rep["status"] == 0 and rep["solver_cluster"] == 0
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    prm = oracle_params(ctx.params, lm=1, lm_mu0=1e-3, gn_iters=G)
    Ro, Eo, nao, acco = O.register(prm, pb, fr, with_accepted=True)
    ties = _check_lm(rep, Eo, acco, G)
    if cfg == "c1":
        assert (acco == 0).any() and (rep["accepted"] == 0).any()
    if not ties:
        terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
        rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
        assert terr.max() < 0.01 and rerr.max() < 1e-4, (terr.max(), rerr.max())


@pytest.mark.parametrize("cfg,G", [("c1", 8), ("c2", 5)])
def test_lm_joint_pose_parity(cfg, G):
    """LM with the joint global pose (the paper's optimiser over nodes + pose)."""
    from tests.test_gpu_pose import joint_ctx, ofr, perturbed_pose
    sc, pb, fr, _ = scene_problem(cfg)
    prior = perturbed_pose(np.array(fr.s.pose[:]))
    ctx, sc2 = joint_ctx(sc, pb, prior, gn_iters=G, flags=M.MIS_F_LM)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert rep["status"] == 0
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    pg = M.mis_get_pose(ctx.ptr)
    prm = oracle_params(ctx.params, lm=1, lm_mu0=1e-3, gn_iters=G, joint_pose=1, w_r=ctx.params.w_r,
                        w_p=ctx.params.w_p)
    Ro, po, Eo, nao, acco = O.register_pose(prm, pb, ofr(sc2), with_accepted=True)
    ties = _check_lm(rep, Eo, acco, G, tot=6)
    if not ties:
        terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
        rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
        assert terr.max() < 0.01 and rerr.max() < 1e-4, (terr.max(), rerr.max())
        assert np.linalg.norm(pg[9:] - po[9:]) < 0.01 and np.abs(pg[:9] - po[:9]).max() < 1e-4


@pytest.mark.parametrize("cfg,G", [("c1", 8), ("c2", 5)])
def test_lm_affine_parity(cfg, G):
    """LM with affine nodes + E_rot (the paper's optimiser over the paper's node model)."""
    from tests.test_gpu_affine import aff_ctx, oprm
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = aff_ctx(sc, pb, flags=M.MIS_F_LM, gn_iters=G)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert rep["status"] == 0
    m = pb.g.shape[0]
    Ag = M.mis_get_nodes_f64(ctx.ptr, m)
    prm = oracle_params(ctx.params, lm=1, lm_mu0=1e-3, gn_iters=G, w_rot=ctx.params.w_rot)
    Ao, Eo, nao, acco = O.register_aff(prm, pb, fr, with_accepted=True)
    ties = _check_lm(rep, Eo, acco, G, tot=5)
    if not ties:
        assert np.linalg.norm(Ag[:, 9:] - Ao[:, 9:], axis=1).max() < 0.01
        assert np.abs(Ag[:, :9] - Ao[:, :9]).max() < 3e-4   # A46
