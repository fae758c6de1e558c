"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Every test here checks the oracle against something other than itself: the
worked examples of tests/golden/spec_examples.json (hand-derived values, each
cited), closed forms, invariants (identity / rigid fields), brute force on tiny
inputs, finite differences, dense linear algebra (numpy) and textbook special
cases.  SURVEY §8(c) "Pins" P1-P16; DESIGN.md §4.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_1803_02009_b200 import synth
from tests.common import apply_perturbation, pose12, random_state, rot, scene_problem

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ helpers
def plane_frame(W=64, H=48, z=50.0, f=40.0, tilt=None):
    """Depth map of a plane seen by the identity camera (analytic ray/plane)."""
    intr = dict(fx=f, fy=f, cx=W / 2.0, cy=H / 2.0, W=W, H=H)
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    if tilt is None:
        D = np.full((H, W), z)
    else:   # plane z = z0 + tan(tilt) * y (about the x axis)
        s = np.tan(np.deg2rad(tilt))
        D = z / (1.0 - s * (v - intr["cy"]) / f)
    return D.astype(np.float32), intr


def single_node_problem(pts, nrms):
    """Every point bound to node 0 (k=1); nodes: 0 at origin and 1 far away."""
    n = len(pts)
    g = np.array([[0, 0, 50.0], [1000, 0, 50.0]], np.float32)
    return O.Problem(np.asarray(pts, np.float32), np.asarray(nrms, np.float32),
                     np.zeros((n, 1), np.int32), np.ones((n, 1), np.float32),
                     g, np.array([[1], [0]], np.int32))


# ------------------------------------------------------------------ P5 projection
def test_p5_projection_golden():
    gp = GOLD["projection"]
    it = gp["intr"]
    D = np.full((it["H"], it["W"]), 50.0, np.float32)
    fr = O.Frame(D, it, pose12())
    pts = np.array([c["point"] for c in gp["cases"]])
    pb = single_node_problem(pts, [[0, 0, -1]] * len(pts))
    prm = O.params(k=1, n_nbr=1)
    pix, why, _ = O.associate(prm, pb, fr, O.identity_state(2))
    for c, p, wb in zip(gp["cases"], pix, why):
        assert wb == 63
        assert p == c["pixel"][1] * it["W"] + c["pixel"][0]
    # back-projection inverse: q at (420, 240) with D=50 is (10, 0, 50)
    q, N, dv, nv = O.frame_prep(fr)
    assert np.allclose(q[240, 420], [10, 0, 50], atol=1e-12)
    assert np.allclose(q[240, 320], [0, 0, 50], atol=1e-12)


def test_p5_roundtrip_random_pixels():
    rng = np.random.default_rng(5)
    D, it = plane_frame(W=97, H=61, f=73.0)
    D = rng.uniform(40, 70, D.shape).astype(np.float32)
    fr = O.Frame(D, it, pose12())
    q, _, _, _ = O.frame_prep(fr)
    ys, xs = rng.integers(0, 61, 100), rng.integers(0, 97, 100)
    Q = q[ys, xs]
    u = it["fx"] * Q[:, 0] / Q[:, 2] + it["cx"]
    v = it["fy"] * Q[:, 1] / Q[:, 2] + it["cy"]
    assert np.max(np.abs(u - xs)) < 1e-9 and np.max(np.abs(v - ys)) < 1e-9


# ------------------------------------------------------------------ P11 normals
def test_p11_normals_plane_and_45deg():
    D, it = plane_frame()
    _, N, dv, nv = O.frame_prep(O.Frame(D, it, pose12()))
    assert nv[1:-1, 1:-1].all() and not nv[0].any() and not nv[:, -1].any()
    assert np.allclose(N[nv], [0, 0, -1], atol=1e-12)
    D45, it = plane_frame(tilt=45.0, z=50.0, f=60.0)
    _, N, _, nv = O.frame_prep(O.Frame(D45, it, pose12()))
    expect = np.array([0.0, 1.0, -1.0]) / np.sqrt(2)   # plane z - y = 50, facing the camera
    err = np.abs(N[nv] - expect).max()
    assert err < GOLD["normals"]["tol_45"], err


def test_p11_hole_neighbour_invalid():
    D, it = plane_frame()
    D[10, 10] = 0.0
    _, _, dv, nv = O.frame_prep(O.Frame(D, it, pose12()))
    assert not dv[10, 10]
    for y, x in [(10, 10), (9, 10), (11, 10), (10, 9), (10, 11)]:
        assert not nv[y, x]
    assert nv[8, 10] and nv[10, 12]


# ------------------------------------------------------------------ P4 skinning
def test_p4_skinning_golden():
    for c in GOLD["skinning"]["cases"]:
        idx, w, _ = O.skin(np.array([c["v"]]), np.array(c["nodes"]), c["k"])
        got = {int(i): float(x) for i, x in zip(idx[0], w[0])}
        exp = {int(a): b for a, b in c["weights"].items()}
        assert set(got) == set(exp)
        for a in exp:
            assert abs(got[a] - exp[a]) < 1e-9


def test_p4_skinning_sum_and_brute_force():
    rng = np.random.default_rng(4)
    g = rng.uniform(-20, 20, (37, 3)).astype(np.float32)
    p = rng.uniform(-20, 20, (200, 3)).astype(np.float32)
    for k in (1, 4, 8):
        idx, w, _ = O.skin(p, g, k)
        assert np.allclose(w.sum(1), 1.0, atol=1e-12)
        assert (w >= 0).all()
        d = np.linalg.norm(p[:, None, :].astype(np.float64) - g[None].astype(np.float64), axis=-1)
        order = np.argsort(d, axis=1, kind="stable")
        assert (np.sort(idx, 1) == np.sort(order[:, :k], 1)).all()
        dk = np.take_along_axis(d, order[:, k:k + 1], 1)
        raw = 1 - np.take_along_axis(d, idx, 1) / dk
        assert np.allclose(w, raw / raw.sum(1, keepdims=True), atol=1e-12)


# ------------------------------------------------------------------ P13 exponential map
def test_p13_exp():
    assert np.array_equal(O.exp_so3([0, 0, 0]), np.eye(3))
    R = O.exp_so3([0, 0, np.pi / 2])
    assert np.allclose(R, [[0, -1, 0], [1, 0, 0], [0, 0, 1]], atol=1e-15)
    rng = np.random.default_rng(13)
    for _ in range(50):
        R = O.exp_so3(rng.normal(0, 1, 3))
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-12)
        assert abs(np.linalg.det(R) - 1) < 1e-12
    w = np.array([3e-13, -1e-13, 2e-13])     # below the first-order switch
    assert np.allclose(O.exp_so3(w), np.eye(3) + np.array(
        [[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]]), atol=1e-24)


# ------------------------------------------------------------------ P1 identity / warp golden
def test_p1_identity_field_leaves_model_unchanged():
    sc, pb, fr, _ = scene_problem("c1")
    xh, nh, vt, nt, ok = O.warp(pb, O.identity_state(pb.g.shape[0]), pose12())
    assert ok.all()
    assert np.abs(vt - pb.xyz).max() < 1e-12
    n64 = pb.nrm.astype(np.float64)
    assert np.abs(nt - n64 / np.linalg.norm(n64, axis=1, keepdims=True)).max() < 1e-12


def test_warp_golden():
    for c in GOLD["warp"]["cases"]:
        pb = single_node_problem([c["v"]], [[1, 0, 0]])
        Rt = O.identity_state(2)
        Rt[0, 9:] = c["t_node"]
        pb.g[0] = 0.0   # node at the origin
        pb = O.Problem(pb.xyz, pb.nrm, pb.idx, pb.w, np.array([[0, 0, 0], [1000, 0, 0]], np.float32), pb.nbr)
        _, _, vt, _, _ = O.warp(pb, Rt, pose12(c["pose_R"], c["pose_T"]))
        assert np.allclose(vt[0], c["out"], atol=1e-12)
    for c in GOLD["normal_warp"]["cases"]:
        pb = single_node_problem([[1, 2, 3]], [c["n"]])
        _, _, _, nt, _ = O.warp(pb, O.identity_state(2), pose12(c["pose_R"]))
        assert np.allclose(nt[0], c["out"], atol=1e-12)


def test_rigid_consistent_field_is_rigid_map():
    """A_j = Q, t_j = (Q-I) g_j + c for all j  =>  warp(v) = R (Q v + c) + T."""
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    Q = rot([1, 2, 3], 7.0)
    c = np.array([1.0, -2.0, 0.5])
    Rt = np.zeros((m, 12))
    for j in range(m):
        Rt[j, :9] = Q.ravel()
        Rt[j, 9:] = (Q - np.eye(3)) @ pb.g[j].astype(np.float64) + c
    R, T = rot([0, 1, 1], 20.0), np.array([3.0, 1.0, -2.0])
    _, _, vt, nt, ok = O.warp(pb, Rt, pose12(R, T))
    v = pb.xyz.astype(np.float64)
    assert np.abs(vt - ((v @ Q.T + c) @ R.T + T)).max() < 1e-9
    n = pb.nrm.astype(np.float64)
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    assert np.abs(nt - n @ Q.T @ R.T).max() < 1e-9


# ------------------------------------------------------------------ P3 regulariser
def _reg_only_system(g, nbr, Rt, w_reg=1.0):
    g = np.asarray(g, np.float32)
    pb = O.Problem(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 1), np.int32), np.zeros((0, 1)),
                   g, np.asarray(nbr, np.int32))
    D, it = plane_frame()
    prm = O.params(k=1, n_nbr=np.asarray(nbr).shape[1], w_reg=w_reg)
    return O.system(prm, pb, O.Frame(D, it, pose12()), Rt)


def test_p3_two_node_golden():
    gr = GOLD["regulariser"]
    Rt = O.identity_state(2)
    Rt[:, 9:] = gr["t"]
    s = _reg_only_system(gr["nodes"], [[1], [0]], Rt)
    assert abs(s["energy"][2] - gr["E_reg"]) < 1e-12


def test_p3_rigid_consistent_reg_is_zero():
    rng = np.random.default_rng(3)
    g = rng.uniform(-30, 30, (40, 3))
    nbr = synth.node_graph(g.astype(np.float32), 4)
    Q = rot([0.3, -1, 2], 25.0)
    c = np.array([4.0, 5.0, -6.0])
    Rt = np.zeros((40, 12))
    for j in range(40):
        Rt[j, :9] = Q.ravel()
        Rt[j, 9:] = (Q - np.eye(3)) @ g[j].astype(np.float32).astype(np.float64) + c
    s = _reg_only_system(g, nbr, Rt)
    assert s["energy"][2] < 1e-18
    assert np.abs(s["rhs"]).max() < 1e-8


# ------------------------------------------------------------------ P8 data term
def test_p8_plane_residual_and_tangential_invariance():
    gd = GOLD["data_term"]
    D, it = plane_frame(z=gd["plane_z"])
    fr = O.Frame(D, it, pose12())
    prm = O.params(k=1, n_nbr=1, w_pt=0.0, w_reg=0.0)
    for x in (0.0, 1.0, 0.37):   # 1 mm tangential shift
        pb = single_node_problem([[x, 0, gd["point_z"]]], [[0, 0, -1]])
        s = O.system(prm, pb, fr, O.identity_state(2))
        assert s["n_assoc"] == 1
        assert abs(np.sqrt(s["energy"][0]) - gd["abs_residual"]) < 1e-9


def test_visibility_golden():
    gv = GOLD["visibility"]
    D, it = plane_frame(z=50.0)
    fr = O.Frame(D, it, pose12())
    prm = O.params(k=1, n_nbr=1, eps_d=gv["eps_d"], eps_n_deg=gv["eps_n_deg"])
    n_tilt = rot([1, 0, 0], gv["tilt_deg"]) @ np.array([0, 0, -1.0])
    n_ok = rot([1, 0, 0], 5.0) @ np.array([0, 0, -1.0])
    pts = [[0, 0, 50 + gv["offset_mm"]], [0, 0, 50 + 10.0], [0, 0, 50.0], [0, 0, 50.0]]
    nrm = [[0, 0, -1], [0, 0, -1], n_tilt, n_ok]
    pb = single_node_problem(pts, nrm)
    pix, why, _ = O.associate(prm, pb, fr, O.identity_state(2))
    assert why[0] == 15 and pix[0] == -1          # 20 mm > eps_d: distance gate fails
    assert why[1] == 63 and pix[1] >= 0
    assert why[2] == 31 and pix[2] == -1          # 15 deg > eps_n: angle gate fails
    assert why[3] == 63


# ------------------------------------------------------------------ P9 association brute force
def _brute_force_association(prm, pb, fr, Rt, intr):
    """Every point against every pixel: the pixel whose unit square (centred on
    the integer coordinate) contains the projection, then the Eq. 7 gates."""
    _, _, vt, nt, ok = O.warp(pb, Rt, np.array(fr.s.pose[:]))
    q, N, dv, nv = O.frame_prep(fr)
    H, W = fr.depth.shape
    xs, ys = np.meshgrid(np.arange(W), np.arange(H))
    out = np.full(len(vt), -1)
    ce = np.cos(np.deg2rad(prm.eps_n_deg))
    for i in range(len(vt)):
        if not ok[i] or vt[i, 2] <= 0:
            continue
        u = intr["fx"] * vt[i, 0] / vt[i, 2] + intr["cx"]
        v = intr["fy"] * vt[i, 1] / vt[i, 2] + intr["cy"]
        hit = (xs - 0.5 <= u) & (u < xs + 0.5) & (ys - 0.5 <= v) & (v < ys + 0.5)
        hit &= dv & nv
        hit &= np.linalg.norm(q - vt[i], axis=-1) < prm.eps_d
        hit &= (N @ nt[i]) > ce
        cand = np.flatnonzero(hit.ravel())
        assert len(cand) <= 1
        if len(cand):
            out[i] = cand[0]
    return out


@pytest.mark.parametrize("seed", range(6))
def test_p9_association_equals_brute_force(seed):
    rng = np.random.default_rng(900 + seed)
    W, H = int(rng.integers(12, 33)), int(rng.integers(12, 33))
    f = float(rng.uniform(15, 30))
    intr = dict(fx=f, fy=f * rng.uniform(0.9, 1.1), cx=W / 2 + rng.uniform(-1, 1), cy=H / 2 + rng.uniform(-1, 1), W=W, H=H)
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    D = (50 + 3 * np.sin(0.3 * u) * np.cos(0.2 * v) + rng.normal(0, 0.3, u.shape)).astype(np.float32)
    D[rng.uniform(size=D.shape) < 0.05] = 0.0
    fr = O.Frame(D, intr, pose12(rot(rng.normal(size=3), 2.0), rng.normal(0, 0.5, 3)))
    n = 300
    pts = np.stack([rng.uniform(-15, 15, n), rng.uniform(-15, 15, n), rng.uniform(45, 56, n)], -1)
    nrm = rng.normal(0, 0.15, (n, 3)) + [0, 0, -1]
    g = rng.uniform(-15, 15, (9, 3)) + [0, 0, 50]
    idx, w, _ = O.skin(pts, g, 3)
    pb = O.Problem(pts, nrm, idx, w, g, synth.node_graph(g.astype(np.float32), 3))
    Rt = random_state(9, rng, 0.02, 0.3)
    prm = O.params(k=3, n_nbr=3)
    pix, why, mg = O.associate(prm, pb, fr, Rt)
    bf = _brute_force_association(prm, pb, fr, Rt, intr)
    keep = mg > 1e-6
    assert (pix[keep] == bf[keep]).all()
    assert (pix >= 0).sum() > 20


# ------------------------------------------------------------------ P6 finite differences
def _small_problem(seed):
    """10 points bound to 4 nodes (k=3) + 2 features on the C1 scene."""
    rng = np.random.default_rng(600 + seed)
    sc = synth.make_scene("c1", 1)
    g_all = sc["g"].astype(np.float64)
    c0 = np.argsort(np.linalg.norm(g_all[:, :2], axis=1))[:4]
    g = sc["g"][c0]
    centre = g.astype(np.float64).mean(0)
    d = np.linalg.norm(sc["xyz"][:, :2] - centre[:2], axis=1)
    near = np.argsort(d)[:400]
    sel = rng.choice(near, 10, replace=False)
    fs = rng.choice(near, 2, replace=False)
    idx, w, _ = O.skin(sc["xyz"][sel], g, 3)
    nbr = synth.node_graph(g, 3)
    fdst = sc["xyz"][fs] @ sc["pose"][:9].reshape(3, 3).T.astype(np.float32) + sc["pose"][9:] + rng.normal(0, 1, (2, 3))
    pb = O.Problem(sc["xyz"][sel], sc["nrm"][sel], idx, w, g, nbr, sc["xyz"][fs], fdst)
    fr = O.Frame(sc["depth"], sc["intr"], sc["pose"])
    prm = O.params(k=3, n_nbr=3, w_pt=1.0)
    return prm, pb, fr, random_state(4, rng, 0.02, 0.3)


def _fd_check(prm, pb, fr, Rt, h=1e-5):
    pix, _, _ = O.associate(prm, pb, fr, Rt)
    fsk = O.feature_skin(pb)[:2]
    r0, J = O.residuals(prm, pb, fr, Rt, pix, fsk)
    m = pb.g.shape[0]
    Jfd = np.zeros_like(J)
    for j in range(m):
        for c in range(6):
            rp, _ = O.residuals(prm, pb, fr, apply_perturbation(Rt, j, c, h), pix, fsk)
            rm, _ = O.residuals(prm, pb, fr, apply_perturbation(Rt, j, c, -h), pix, fsk)
            Jfd[:, 6 * j + c] = (rp - rm) / (2 * h)
    return J, Jfd, pix


@pytest.mark.parametrize("seed", range(20))
def test_p6_finite_difference_jacobians_small(seed):
    prm, pb, fr, Rt = _small_problem(seed)
    J, Jfd, pix = _fd_check(prm, pb, fr, Rt)
    assert (pix >= 0).sum() >= 5
    rel = np.abs(J - Jfd).max() / np.abs(J).max()
    assert rel < 1e-4, rel


def test_p6_finite_difference_jacobians_c1():
    sc, pb, fr, _ = scene_problem("c1")
    sub = np.random.default_rng(61).choice(pb.xyz.shape[0], 300, replace=False)
    pb = O.Problem(pb.xyz[sub], pb.nrm[sub], pb.idx[sub], pb.w[sub], pb.g, pb.nbr, pb.fsrc, pb.fdst)
    Rt = random_state(pb.g.shape[0], np.random.default_rng(62), 0.01, 0.3)
    prm = O.params()
    J, Jfd, pix = _fd_check(prm, pb, fr, Rt)
    rel = np.abs(J - Jfd).max() / np.abs(J).max()
    assert rel < 1e-4, rel


# ------------------------------------------------------------------ P7 / P14 assembly and solves
def test_p7_assembly_equals_dense_jtj_c1():
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    Rt = random_state(m, np.random.default_rng(70), 0.01, 0.3)
    prm = O.params()
    s = O.system(prm, pb, fr, Rt)
    pix, _, _ = O.associate(prm, pb, fr, Rt)
    r, J = O.residuals(prm, pb, fr, Rt, pix)
    Hd = J.T @ J
    H = O.dense_H(s, m)
    scale = np.abs(Hd).max()
    assert np.abs(H - Hd).max() < 1e-10 * scale
    assert np.abs(s["rhs"] + J.T @ r).max() < 1e-10 * np.abs(J.T @ r).max()
    assert abs(s["energy"][4] - r @ r) < 1e-10 * (r @ r)
    # P14: symmetric positive semi-definite
    ev = np.linalg.eigvalsh(0.5 * (H + H.T))
    assert ev.min() > -1e-10 * ev.max()
    assert s["n_assoc"] == int((pix >= 0).sum())


def test_p7_solves_match_dense():
    sc, pb, fr, _ = scene_problem("c2", with_features=True)
    m = pb.g.shape[0]
    prm = O.params()
    s = O.system(prm, pb, fr, O.identity_state(m))
    A = O.dense_H(s, m) + prm.lambda_ * np.eye(6 * m)
    x_ref = np.linalg.solve(A, s["rhs"])
    x, _ = O.solve(s, m, prm.lambda_, 0, 0)          # EXACT (PCG to 1e-12 at this size)
    assert np.abs(A @ x - s["rhs"]).max() < 1e-9 * np.abs(s["rhs"]).max()
    assert np.abs(x - x_ref).max() < 1e-6 * np.abs(x_ref).max()
    # MIRROR, one iteration = preconditioned steepest descent from 0: x = (b.z)/(z.A z) z, z = M b
    Minv = np.zeros((6 * m, 6 * m))
    Hd = O.dense_H(s, m)
    for j in range(m):
        B = Hd[6 * j:6 * j + 6, 6 * j:6 * j + 6]
        mu = 1e-9 * np.trace(B) / 6
        Minv[6 * j:6 * j + 6, 6 * j:6 * j + 6] = np.linalg.inv(B + (prm.lambda_ + mu) * np.eye(6))
    z = Minv @ s["rhs"]
    x1_ref = (s["rhs"] @ z) / (z @ A @ z) * z
    x1, _ = O.solve(s, m, prm.lambda_, 1, 1)
    assert np.abs(x1 - x1_ref).max() < 1e-9 * np.abs(x1_ref).max()


def test_p7_exact_small_is_cholesky():
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    prm = O.params()
    s = O.system(prm, pb, fr, O.identity_state(m))
    A = O.dense_H(s, m) + prm.lambda_ * np.eye(6 * m)
    x, _ = O.solve(s, m, prm.lambda_, 0, 0)
    assert np.abs(x - np.linalg.solve(A, s["rhs"])).max() < 1e-9 * np.abs(x).max()


# ------------------------------------------------------------------ P15 shard invariance
def test_p15_shard_sum_equals_full_system():
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    Rt = random_state(m, np.random.default_rng(150), 0.01, 0.2)
    prm = O.params()
    full = O.system(prm, pb, fr, Rt)
    n = pb.xyz.shape[0]
    cuts = [0, n // 3, 2 * n // 3, n]
    Hs = np.zeros((6 * m, 6 * m)); rhs = np.zeros(6 * m); E = np.zeros(5)
    for s_ in range(3):
        a, b = cuts[s_], cuts[s_ + 1]
        nbr = pb.nbr if s_ == 0 else np.full_like(pb.nbr, -1)   # graph terms on shard 0 only
        fs = (pb.fsrc, pb.fdst) if s_ == 0 else (None, None)
        sb = O.Problem(pb.xyz[a:b], pb.nrm[a:b], pb.idx[a:b], pb.w[a:b], pb.g, nbr, *fs)
        ss = O.system(prm, sb, fr, Rt)
        Hs += O.dense_H(ss, m); rhs += ss["rhs"]; E += ss["energy"]
    Hf = O.dense_H(full, m)
    assert np.abs(Hs - Hf).max() < 1e-10 * np.abs(Hf).max()
    assert np.abs(rhs - full["rhs"]).max() < 1e-10 * np.abs(full["rhs"]).max()
    assert np.allclose(E, full["energy"], rtol=1e-12)


# ------------------------------------------------------------------ P2 / P12 rigid recovery
def _rigid_scene(Q, c, cfg="c1", n_feat=24, bump=True):
    """Noise-free observation of the frame-0 surface after a rigid tissue motion
    (Q, c), seen by the identity camera (PAPER.md:616 protocol without noise)."""
    cfgo = synth.CONFIGS[cfg]
    rng = np.random.default_rng(20)
    bumps = [(3.0, -2.0, 2.5, synth.BUMP_SIGMA)] if bump else []
    surf = synth.Surface(0.0, bumps)
    mdl = synth.sample_model(cfgo, surf, rng, 0)
    # tissue motion (Q, c) in world == camera pose (Q, c) on the unmoved tissue
    depth = synth.render_depth(cfgo, surf, Q, c, rng, noise=False, holes=False)
    idx, w, _ = O.skin(mdl["xyz"], mdl["g"], cfgo.k)
    fsel = rng.choice(len(mdl["xyz"]), n_feat, replace=False)
    fsrc = mdl["xyz"][fsel]
    fdst = fsrc.astype(np.float64) @ Q.T + c
    pb = O.Problem(mdl["xyz"], mdl["nrm"], idx, w, mdl["g"], mdl["nbr"], fsrc, fdst)
    fr = O.Frame(depth, synth.intrinsics(cfgo), pose12())
    return pb, fr


@pytest.mark.parametrize("Qc", [
    (rot([0, 0, 1], 0.0), np.array([2.0, 0.0, 0.0])),          # S:294 pure translation (2,0,0)
    (rot([1, -2, 0.5], 1.5), np.array([0.8, -0.5, 0.6])),      # general rigid motion
])
def test_p2_rigid_motion_recovered(Qc):
    Q, c = Qc
    pb, fr = _rigid_scene(Q, c)
    m = pb.g.shape[0]
    prm = O.params(w_pt=0.0, gn_iters=8, solve_mode=0)
    Rt, E, na = O.register(prm, pb, fr)
    g = pb.g.astype(np.float64)
    t_exp = g @ (Q - np.eye(3)).T + c
    terr = np.linalg.norm(Rt[:, 9:] - t_exp, axis=1)
    rerr = np.array([np.linalg.norm(_log(Rt[j, :9].reshape(3, 3) @ Q.T)) for j in range(m)])
    assert terr.max() < 0.01, terr.max()
    assert rerr.max() < 1e-4, rerr.max()
    assert E[-1, 4] < 1e-3 * E[0, 4]


def _log(R):
    c = np.clip((np.trace(R) - 1) / 2, -1, 1)
    th = np.arccos(c)
    if th < 1e-9:
        return np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]]) / 2
    return th / (2 * np.sin(th)) * np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])


def test_p12_fixed_point():
    pb, fr = _rigid_scene(np.eye(3), np.zeros(3))
    prm = O.params(w_pt=0.0, gn_iters=6, solve_mode=0)
    Rt, E, _ = O.register(prm, pb, fr)
    prm1 = O.params(w_pt=0.0, gn_iters=1, solve_mode=0)
    Rt2, E2, _ = O.register(prm1, pb, fr, Rt)
    assert abs(E2[1, 4] - E2[0, 4]) < 1e-10 * max(1.0, E2[0, 4])
    assert np.abs(Rt2 - Rt).max() < 1e-6


def test_p16_energy_non_increasing_noiseless():
    """Sanity (not a gate): fixed-P (MIRROR) GN on a noise-free, exactly
    representable deformation (a rigid tissue motion) lowers the energy every
    iteration.  (A 2-3 mm bump is NOT representable by C1's 16 nodes, and
    point-to-plane alone leaves near-null modes on the bowl, so those are not
    used here.)"""
    pb, fr = _rigid_scene(rot([0.2, 1, -0.4], 1.0), np.array([0.5, 0.3, -0.4]))
    Rt, E, na = O.register(O.params(w_pt=0.0, gn_iters=5, pcg_iters=10, solve_mode=1), pb, fr)
    tot = E[:, 4]
    assert (np.diff(tot) <= 1e-9 * tot[0]).all(), tot
    assert tot[-1] < 0.25 * tot[0]   # 10 PCG iterations do not fully converge


# ------------------------------------------------------------------ P10 fusion
def test_p10_fusion_golden_and_cap():
    gf = GOLD["fusion"]
    D, it = plane_frame(z=gf["depth"], f=40.0)
    fr = O.Frame(D, it, pose12())
    prm = O.params(k=1, n_nbr=1, tau_z=10.0, trunc=40.0)
    xyz = np.array([[0, 0, gf["model_z"]], [0.3, 0.0, gf["model_z"] + 0.5]], np.float32)
    # second point lands on another pixel; give it omega = omega_max
    xyz[1] = [12.0 / 40 * 10.0 * 2, 0, gf["model_z"]]
    nrm = np.array([[0, 0, -1], [0, 0, -1]], np.float32)
    rgb = np.zeros((2, 3), np.float32)
    out = O.fuse(prm, xyz, nrm, rgb, np.array([gf["omega"], prm.omega_max], np.float32),
                 np.zeros(2, np.int32), fr, None, 7, np.array([[0, 0, 0], [100, 0, 0]], np.float32))
    assert abs(out["xyz"][0, 2] - gf["fused_z"]) < 1e-12
    assert out["weight"][0] == 2.0 and out["stamp"][0] == 7
    assert out["weight"][1] == prm.omega_max
    assert (out["weight"] <= prm.omega_max).all()


def _fusion_scene(seed, W=32, H=24):
    rng = np.random.default_rng(1000 + seed)
    f = 30.0
    intr = dict(fx=f, fy=f, cx=W / 2, cy=H / 2, W=W, H=H)
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    D = (50 + 2 * np.sin(0.25 * u + 0.1 * v)).astype(np.float32)
    D[rng.uniform(size=D.shape) < 0.04] = 0.0
    fr = O.Frame(D, intr, pose12(rot(rng.normal(size=3), 1.0), rng.normal(0, 0.3, 3)))
    n = 900
    pts = np.stack([rng.uniform(-25, 25, n), rng.uniform(-19, 19, n), rng.uniform(45, 57, n)], -1).astype(np.float32)
    nrm = (rng.normal(0, 0.1, (n, 3)) + [0, 0, -1]).astype(np.float32)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return fr, intr, pts, nrm, rng


@pytest.mark.parametrize("seed", range(4))
def test_p10_registration_brute_force_and_accounting(seed):
    fr, intr, pts, nrm, rng = _fusion_scene(seed)
    n = len(pts)
    prm = O.params(k=2, n_nbr=1)
    g = rng.uniform(-20, 20, (6, 3)).astype(np.float32) + np.float32([0, 0, 50])
    out = O.fuse(prm, pts, nrm, rng.uniform(0, 1, (n, 3)), rng.integers(1, 11, n).astype(np.float32),
                 np.zeros(n, np.int32), fr, rng.uniform(0, 1, (intr["H"], intr["W"], 3)), 3, g)
    # brute force: every point against every pixel, same gates, lexicographic (|dz|, i) min
    q, N, dv, nv = O.frame_prep(fr)
    pose = np.array(fr.s.pose[:])
    R, T = pose[:9].reshape(3, 3), pose[9:]
    vt = pts.astype(np.float64) @ R.T + T
    nt = nrm.astype(np.float64) @ R.T
    H, W = fr.depth.shape
    xs, ys = np.meshgrid(np.arange(W), np.arange(H))
    best = {}
    cd = np.cos(np.deg2rad(prm.delta_deg))
    for i in range(n):
        if vt[i, 2] <= 0:
            continue
        u = intr["fx"] * vt[i, 0] / vt[i, 2] + intr["cx"]
        v = intr["fy"] * vt[i, 1] / vt[i, 2] + intr["cy"]
        hit = (xs - 0.5 <= u) & (u < xs + 0.5) & (ys - 0.5 <= v) & (v < ys + 0.5) & dv & nv
        dz = np.abs(vt[i, 2] - fr.depth.astype(np.float64))
        hit &= (dz < min(prm.tau_z, prm.trunc)) & ((N @ nt[i]) > cd)
        for p in np.flatnonzero(hit.ravel()):
            key = (dz.ravel()[p], i)
            if p not in best or key < best[p]:
                best[p] = key
    owner = out["owner"]
    for p in range(H * W):
        if out["key_margin"][p] <= 1e-6:
            continue
        assert owner[p] == (best[p][1] if p in best else -1)
    # pixel accounting: every valid pixel is registered once or lifted once
    valid = (dv & nv).ravel()
    assert (owner >= 0).sum() + out["n_lift"] == valid.sum()
    assert len(set(owner[owner >= 0])) == (owner >= 0).sum()
    assert (out["weight"] <= prm.omega_max).all()
    assert out["lift_w"].shape[0] == out["n_lift"] and np.allclose(out["lift_w"].sum(1), 1.0)


def test_p10_refuse_contracts():
    """Fusing the identical scan twice moves points less the second time."""
    fr, intr, pts, nrm, rng = _fusion_scene(7)
    n = len(pts)
    prm = O.params(k=2, n_nbr=1)
    g = np.array([[0, 0, 50], [10, 0, 50], [0, 10, 50]], np.float32)
    w0 = np.ones(n, np.float32)
    o1 = O.fuse(prm, pts, nrm, np.zeros((n, 3)), w0, np.zeros(n, np.int32), fr, None, 1, g)
    x1 = o1["xyz"][:n].astype(np.float32)
    o2 = O.fuse(prm, x1, o1["nrm"][:n], np.zeros((n, 3)), o1["weight"][:n], np.zeros(n, np.int32), fr, None, 2, g)
    d1 = np.linalg.norm(o1["xyz"][:n] - pts, axis=1)
    d2 = np.linalg.norm(o2["xyz"][:n] - x1, axis=1)
    moved = d1 > 1e-9
    assert moved.sum() > 50
    assert d2[moved].sum() < d1[moved].sum()


# ------------------------------------------------------------------ more closed forms
def test_point_to_point_and_feature_residuals_golden():
    """r_pt = v~ - q (north_star point-to-point) on the S:214 plane example; E_corr
    (Eq. 9): identity field and V = V' -> 0, global T = (1,0,0) -> (1,0,0) per pair."""
    gd = GOLD["data_term"]
    D, it = plane_frame(z=gd["plane_z"])
    fr = O.Frame(D, it, pose12())
    pb = single_node_problem([[0, 0, gd["point_z"]]], [[0, 0, -1]])
    s = O.system(O.params(k=1, n_nbr=1, w_reg=0.0), pb, fr, O.identity_state(2))
    assert abs(s["energy"][1] - 4.0) < 1e-12     # |(0,0,2)|^2
    src = np.array([[1.0, 2.0, 50.0], [-3.0, 0.5, 48.0]], np.float32)
    g = np.array([[0, 0, 50], [5, 0, 50], [0, 5, 50]], np.float32)
    for T, e in [(np.zeros(3), 0.0), (np.array([1.0, 0, 0]), 2.0)]:
        pb = O.Problem(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 2), np.int32), np.zeros((0, 2)),
                       g, np.array([[1], [0], [0]], np.int32), src, src)
        s = O.system(O.params(k=2, n_nbr=1, w_reg=0.0), pb, O.Frame(D, it, pose12(None, T)), O.identity_state(3))
        assert abs(s["energy"][3] - e) < 1e-12


def test_warp_model_closed_forms():
    """O4: identity field -> unchanged model; rigid-consistent field -> rigid map;
    nodes advance by t_j (R-A26)."""
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    xyz, nrm, g = O.warp_model(pb, O.identity_state(m))
    assert np.abs(xyz - pb.xyz).max() < 1e-12 and np.abs(g - pb.g).max() < 1e-12
    Q, c = rot([1, 0, 1], 5.0), np.array([0.5, -1.0, 2.0])
    Rt = np.zeros((m, 12))
    Rt[:, :9] = Q.ravel()
    Rt[:, 9:] = pb.g.astype(np.float64) @ (Q - np.eye(3)).T + c
    xyz, nrm, g = O.warp_model(pb, Rt)
    assert np.abs(xyz - (pb.xyz.astype(np.float64) @ Q.T + c)).max() < 1e-9
    n64 = pb.nrm.astype(np.float64)
    assert np.abs(nrm - (n64 / np.linalg.norm(n64, axis=1, keepdims=True)) @ Q.T).max() < 1e-9
    assert np.abs(g - (pb.g.astype(np.float64) + Rt[:, 9:])).max() < 1e-12


def test_fusion_colour_normal_golden():
    """Eq. 13: omega=1, C=0, C_obs=1 -> 0.5; Eq. 14: equal normals stay; lifted
    point = back-projected pixel with omega=1, stamp=frame (Alg. 2 Step 3)."""
    D, it = plane_frame(z=12.0, f=40.0)
    fr = O.Frame(D, it, pose12())
    prm = O.params(k=1, n_nbr=1)
    xyz = np.array([[0, 0, 10.0]], np.float32)
    out = O.fuse(prm, xyz, np.array([[0, 0, -1]], np.float32), np.zeros((1, 3), np.float32),
                 np.ones(1, np.float32), np.zeros(1, np.int32), fr,
                 np.ones((it["H"], it["W"], 3), np.float32), 4, np.array([[0, 0, 0], [9, 9, 9]], np.float32))
    assert np.allclose(out["rgb"][0], 0.5, atol=1e-12)
    assert np.allclose(out["nrm"][0], [0, 0, -1], atol=1e-12)
    valid = (it["W"] - 2) * (it["H"] - 2)
    assert out["n_lift"] == valid - 1
    p = 1 + 0   # first lifted point = pixel (1, 1) in row-major order
    assert np.allclose(out["xyz"][p], [(1 - it["cx"]) * 12 / 40, (1 - it["cy"]) * 12 / 40, 12], atol=1e-12)
    assert out["weight"][p] == 1.0 and out["stamp"][p] == 4 and np.allclose(out["rgb"][p], 1.0)


# ------------------------------------------------------------------ NEXT-3: Levenberg-Marquardt (R-A29)
def _lm_dense(prm, pb, fr, G, mu0):
    """Levenberg-Marquardt written out with dense numpy algebra on the oracle's assembly
    (an independent implementation of the schedule: P:166 LM, S:303 Marquardt damping
    lambda diag(J^T J), x10 on rejection, x0.5 on acceptance; the base lambda I of R-A16)."""
    m = pb.g.shape[0]
    Rt = O.identity_state(m)
    base, acc_sys, E_acc, mu = Rt.copy(), None, 0.0, mu0
    Es, accs = [], []
    for it in range(G + 1):
        s = O.system(prm, pb, fr, Rt)
        E = s["energy"][4]
        ok = it == 0 or E < E_acc
        Es.append(E)
        accs.append(int(ok))
        if ok:
            base, acc_sys, E_acc = Rt.copy(), s, E
            if it > 0:
                mu *= 0.5
        else:
            Rt = base.copy()
            mu *= 10.0
        if it == G:
            break
        H = O.dense_H(acc_sys, m)
        A = H + np.diag(mu * np.diag(H)) + prm.lambda_ * np.eye(6 * m)
        x = np.linalg.solve(A, acc_sys["rhs"])
        Rn = base.copy()
        for j in range(m):
            Rn[j, :9] = (O.exp_so3(x[6 * j:6 * j + 3]) @ base[j, :9].reshape(3, 3)).ravel()
            Rn[j, 9:] = base[j, 9:] + x[6 * j + 3:6 * j + 6]
        Rt = Rn
    return Rt, np.array(Es), np.array(accs)


def test_lm_matches_dense_reimplementation():
    """The oracle's LM loop (EXACT solves) against the dense numpy rewrite: same trial
    energies, same accept / reject decisions (including rejections), same final state."""
    sc, pb, fr, _ = scene_problem("c1")
    G = 8
    prm = O.params(gn_iters=G, solve_mode=0, lm=1, lm_mu0=1e-3)
    Rt, E, na, acc = O.register(prm, pb, fr, with_accepted=True)
    Rd, Ed, accd = _lm_dense(prm, pb, fr, G, 1e-3)
    assert (acc == accd).all(), (acc, accd)
    assert (acc == 0).any() and (acc[1:] == 1).any()   # both branches exercised
    assert np.abs(E[:, 4] - Ed).max() < 1e-9 * Ed[0]
    assert np.abs(Rt - Rd).max() < 1e-9


def test_lm_zero_damping_all_accepted_is_gauss_newton():
    """mu0 = 0 and every trial accepted (GN decreasing here for 2 iterations): LM is GN."""
    sc, pb, fr, _ = scene_problem("c1")
    gn = O.params(gn_iters=2, solve_mode=1)
    lm = O.params(gn_iters=2, solve_mode=1, lm=1, lm_mu0=0.0)
    Rg, Eg, _ = O.register(gn, pb, fr)
    Rl, El, _, acc = O.register(lm, pb, fr, with_accepted=True)
    assert (acc == 1).all()
    assert np.array_equal(Rg, Rl) and np.array_equal(Eg, El)


def test_lm_accepted_energy_strictly_decreasing_and_final_is_best():
    """the accepted energy sequence decreases; the returned state is the last
    accepted one (its energy, re-evaluated, is the minimum of the accepted energies)."""
    sc, pb, fr, _ = scene_problem("c1")
    prm = O.params(gn_iters=10, solve_mode=1, lm=1, lm_mu0=1e-3)
    Rt, E, na, acc = O.register(prm, pb, fr, with_accepted=True)
    ea = E[acc == 1, 4]
    assert (np.diff(ea) < 0).all(), ea
    Ef = O.system(prm, pb, fr, Rt)["energy"][4]
    assert abs(Ef - ea[-1]) < 1e-9 * ea[0]
    assert (E[acc == 0, 4] >= ea.min()).all()


# ------------------------------------------------------------------ O7: Alg. 3 filtering (NEXT-1)
def _flt(xyz, w, stamp, grid, frame=20, tau_time=10, tau_weight=3.0, omega_max=20.0, nrm=None, rgb=None, ids=None):
    xyz = np.asarray(xyz, np.float64)
    n = len(xyz)
    nrm = np.tile([0.0, 0.0, 1.0], (n, 1)) if nrm is None else nrm
    rgb = np.zeros((n, 3)) if rgb is None else rgb
    return O.filter_points(xyz, nrm, rgb, np.asarray(w, np.float64), np.asarray(stamp), ids, grid, frame,
                           tau_time, tau_weight, omega_max)


def test_filter_spec_two_point_cell():
    """one cell, weights 1 and 3, depths 10 and 20 -> weighted mean (10*1 + 20*3)/4 = 17.5, omega 4."""
    o = _flt([[0.5, 0.5, 10.0], [0.5, 0.5, 20.0]], [1.0, 3.0], [20, 20], grid=100.0)
    assert o["cells"] == 1 and len(o["weight"]) == 1
    np.testing.assert_allclose(o["xyz"][0], [0.5, 0.5, 17.5], rtol=0, atol=1e-12)
    assert o["weight"][0] == 4.0 and o["stable"][0] == 1


def test_filter_spec_time_rule():
    """S:373-374 ("time stamp threshold is set to 10"): delete iff t < frame - tau_time and omega < tau_weight."""
    pts = [[0.5, 0.5, 0.5], [10.5, 0.5, 0.5], [20.5, 0.5, 0.5], [30.5, 0.5, 0.5]]
    # fresh (t = frame), last seen tau_time ago (kept: boundary), tau_time+1 ago (deleted), old but heavy (kept)
    o = _flt(pts, [1.0, 1.0, 1.0, 5.0], [20, 10, 9, 0], grid=1.0, frame=20, tau_time=10, tau_weight=3.0)
    np.testing.assert_array_equal(o["xyz"][:, 0], [0.5, 10.5, 30.5])
    np.testing.assert_array_equal(o["stable"], [0, 0, 1])
    np.testing.assert_array_equal(o["ids"], [0, 1, 3])


def test_filter_weight_cap_and_zero_weight_cell():
    """Eq. 15 cap in the merge; a cell whose weights sum to 0 takes the plain mean."""
    o = _flt([[0.2, 0.2, 0.2], [0.4, 0.4, 0.4], [5.1, 5.1, 5.1], [5.3, 5.1, 5.1]], [15.0, 9.0, 0.0, 0.0],
             [20, 20, 20, 20], grid=1.0, omega_max=20.0)
    assert o["weight"][0] == 20.0
    np.testing.assert_allclose(o["xyz"][0], np.full(3, (15 * 0.2 + 9 * 0.4) / 24.0), atol=1e-7)
    np.testing.assert_allclose(o["xyz"][1], [5.2, 5.1, 5.1], atol=1e-6)
    assert o["weight"][1] == 0.0


def test_filter_single_cell_is_weighted_centroid():
    """A box holding every point: numpy's weighted average, renormalised mean normal, max stamp, first id."""
    rng = np.random.default_rng(7)
    n = 50
    xyz = rng.uniform(1.0, 9.0, (n, 3))
    nrm = rng.normal(size=(n, 3)); nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[:, 2] = np.abs(nrm[:, 2]) + 0.5
    rgb = rng.uniform(0, 1, (n, 3))
    w = rng.uniform(0.5, 2.0, n)
    st = rng.integers(0, 20, n)
    ids = rng.integers(1000, 2000, n)
    o = _flt(xyz, w, st, grid=10.0, nrm=nrm, rgb=rgb, ids=ids, omega_max=1e9)
    x32 = xyz.astype(np.float32).astype(np.float64)
    np.testing.assert_allclose(o["xyz"][0], np.average(x32, axis=0, weights=w.astype(np.float32)), rtol=1e-12)
    np.testing.assert_allclose(o["rgb"][0], np.average(rgb.astype(np.float32).astype(np.float64), axis=0,
                                                          weights=w.astype(np.float32)),
                               rtol=1e-12)
    nm = np.average(nrm.astype(np.float32).astype(np.float64), axis=0, weights=w.astype(np.float32))
    np.testing.assert_allclose(o["nrm"][0], nm / np.linalg.norm(nm), rtol=1e-12)
    assert o["stamp"][0] == st.max() and o["ids"][0] == ids[0]
    np.testing.assert_allclose(o["weight"][0], w.astype(np.float32).astype(np.float64).sum(), rtol=1e-12)


def test_filter_distinct_cells_is_a_sorted_identity():
    """Grid finer than the spacing: every point alone -> values unchanged, order = lexsort of the cell keys."""
    rng = np.random.default_rng(3)
    lat = np.stack(np.meshgrid(np.arange(6), np.arange(5), np.arange(4), indexing="ij"), -1).reshape(-1, 3)
    perm = rng.permutation(len(lat))
    xyz = (lat[perm] * 2.0 + 0.5).astype(np.float32)
    w = rng.uniform(1, 5, len(xyz)).astype(np.float32)
    o = _flt(xyz, w, np.full(len(xyz), 20), grid=2.0, omega_max=100.0)
    order = np.lexsort((lat[perm][:, 2], lat[perm][:, 1], lat[perm][:, 0]))
    np.testing.assert_array_equal(o["xyz"], xyz[order].astype(np.float64))
    np.testing.assert_array_equal(o["weight"], w[order].astype(np.float64))
    np.testing.assert_array_equal(o["ids"], order)


def test_filter_conserves_weighted_mass_and_stays_in_cell():
    """Random cloud, no cap, no deletion: per-cell sum of omega*v conserved, merged points inside their box,
    cell count = distinct floor keys (numpy), keys strictly ascending."""
    rng = np.random.default_rng(11)
    n = 4000
    xyz = rng.normal(0, 20, (n, 3)).astype(np.float32)
    w = rng.uniform(0.5, 3.0, n).astype(np.float32)
    grid = np.float32(3.0)
    o = _flt(xyz, w, np.zeros(n, int), grid=float(grid), frame=0, tau_time=10, omega_max=1e9)
    keys = np.floor(xyz / grid).astype(np.int64)
    uk, inv = np.unique(keys, axis=0, return_inverse=True)
    assert o["cells"] == len(uk) == len(o["weight"])
    mass = np.zeros((len(uk), 3)); np.add.at(mass, inv.ravel(), w[:, None].astype(np.float64) * xyz)
    wsum = np.zeros(len(uk)); np.add.at(wsum, inv.ravel(), w.astype(np.float64))
    np.testing.assert_allclose(o["weight"], wsum, rtol=1e-12)
    np.testing.assert_allclose(o["xyz"] * o["weight"][:, None], mass, rtol=1e-9, atol=1e-9)
    ok = np.floor(o["xyz"] / float(grid)).astype(np.int64)
    np.testing.assert_array_equal(ok, uk)   # np.unique sorts lexicographically: the same ascending order


# ------------------------------------------------------------------ Eq. 12-14 and the world back-transform
def test_eq14_unequal_normals_and_back_transform_under_pose():
    """Eq. 12-14 with omega = 3 and unequal normals under a non-identity pose, against geometry
    written in the camera-to-world parametrisation (rotation Rc, centre C; world->camera is then
    R = Rc^T, T = -Rc^T C): a rigid map preserves affine combinations, so the fused world point is
    (omega v + q_w) / (omega + 1) with q_w = C + Rc q; by the law of sines in the parallelogram of
    omega n~ and N the fused normal makes tan(phi) = omega sin(theta) / (1 + omega cos(theta)) with
    N, in their plane, on n~'s side; Eq. 13 colours; lifted pixels (Alg. 2 Step 3) land at
    C + Rc q with normal Rc N.  An R / R^T slip, an unweighted or unnormalised blend or a dropped
    T fails one of these."""
    W, H, f, D = 64, 48, 40.0, 50.0
    it = dict(fx=f, fy=f, cx=W / 2.0, cy=H / 2.0, W=W, H=H)
    depth = np.full((H, W), D, np.float32)            # fronto-parallel in the camera frame: N = (0, 0, -1)
    Rc = rot([1.0, 2.0, -0.5], 25.0)
    C = np.array([3.0, -2.0, 5.0])
    fr = O.Frame(depth, it, pose12(Rc.T, -Rc.T @ C))
    px, py = 40, 30
    q_cam = np.array([(px - it["cx"]) * D / f, (py - it["cy"]) * D / f, D])
    v_cam = q_cam * (47.0 / D)                        # same pixel ray, |dz| = 3 mm < tau_z
    theta = np.deg2rad(8.0)                           # < delta = 10 deg
    n_cam = np.array([0.0, np.sin(theta), -np.cos(theta)])
    omega = 3.0
    xyz = (C + Rc @ v_cam)[None].astype(np.float32)
    nrm = (Rc @ n_cam)[None].astype(np.float32)
    rgb = np.array([[0.2, 0.4, 0.8]], np.float32)
    obs = np.zeros((H, W, 3), np.float32)
    obs[py, px] = [0.6, 0.0, 0.4]
    obs[1, 1] = [0.25, 0.5, 0.75]
    prm = O.params(k=1, n_nbr=1)
    out = O.fuse(prm, xyz, nrm, rgb, np.array([omega], np.float32), np.zeros(1, np.int32), fr, obs, 6,
                 np.array([[0, 0, 50.0], [99, 0, 50.0]], np.float32))
    assert out["owner"][py * W + px] == 0
    v_w = xyz[0].astype(np.float64)
    q_w = C + Rc @ q_cam
    assert np.abs(out["xyz"][0] - (omega * v_w + q_w) / (omega + 1)).max() < 1e-9
    phi = np.arctan2(omega * np.sin(theta), 1 + omega * np.cos(theta))
    assert 0 < phi < theta and abs(phi - theta * omega / (omega + 1)) > 2e-5   # not the angle-weighted mean (slerp)
    n_exp = Rc @ np.array([0.0, np.sin(phi), -np.cos(phi)])
    assert np.abs(out["nrm"][0] - n_exp).max() < 1e-6   # fp32 storage of the input normal
    assert abs(np.linalg.norm(out["nrm"][0]) - 1) < 1e-12
    assert np.allclose(out["rgb"][0], [0.3, 0.3, 0.7], atol=1e-7)
    assert out["weight"][0] == 4.0 and out["stamp"][0] == 6
    # lifted: every valid pixel except the registered one, row-major; the first is (1, 1)
    assert out["n_lift"] == (W - 2) * (H - 2) - 1
    q11 = np.array([(1 - it["cx"]) * D / f, (1 - it["cy"]) * D / f, D])
    assert np.abs(out["xyz"][1] - (C + Rc @ q11)).max() < 1e-9
    assert np.abs(out["nrm"][1] - Rc @ np.array([0, 0, -1.0])).max() < 1e-12
    assert np.allclose(out["rgb"][1], [0.25, 0.5, 0.75]) and out["weight"][1] == 1.0 and out["stamp"][1] == 6
    # the registered pixel is not lifted: no lifted point lies on its ray
    lw = out["xyz"][1:]
    lc = (lw - C) @ Rc                                 # back to the camera frame via Rc^T (x - C)
    u = f * lc[:, 0] / lc[:, 2] + it["cx"]
    v = f * lc[:, 1] / lc[:, 2] + it["cy"]
    assert not np.any((np.abs(u - px) < 1e-6) & (np.abs(v - py) < 1e-6))


# ------------------------------------------------------------------ MIRROR PCG at P = 10 (O3h)
def _textbook_pcg(A, b, Minv, P):
    """Preconditioned CG from x0 = 0, P iterations (Hestenes-Stiefel, Saad Alg. 9.1), dense numpy."""
    x = np.zeros_like(b)
    r = b.copy()
    z = Minv @ r
    p = z.copy()
    rz = r @ z
    for _ in range(P):
        Ap = A @ p
        alpha = rz / (p @ Ap)
        x += alpha * p
        r -= alpha * Ap
        z = Minv @ r
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x


def _block_jacobi(Hd, m, lam):
    Minv = np.zeros_like(Hd)
    for j in range(m):
        B = Hd[6 * j:6 * j + 6, 6 * j:6 * j + 6]
        mu = 1e-9 * np.trace(B) / 6                      # R-A17
        Minv[6 * j:6 * j + 6, 6 * j:6 * j + 6] = np.linalg.inv(B + (lam + mu) * np.eye(6))
    return Minv


def test_mirror_pcg_p10_is_textbook_pcg():
    """O3h MIRROR with the GPU's P = 10 against textbook dense PCG with the block-Jacobi
    preconditioner of R-A17, on the C2 system (P = 10 is far from convergence there, so a wrong
    recurrence -- beta, the residual update, the preconditioner -- shows)."""
    sc, pb, fr, _ = scene_problem("c2")
    m = pb.g.shape[0]
    prm = O.params()
    s = O.system(prm, pb, fr, random_state(m, np.random.default_rng(8), 0.01, 0.3))
    Hd = O.dense_H(s, m)
    A = Hd + prm.lambda_ * np.eye(6 * m)
    Minv = _block_jacobi(Hd, m, prm.lambda_)
    for P in (2, 10):
        x_ref = _textbook_pcg(A, s["rhs"], Minv, P)
        x, it = O.solve(s, m, prm.lambda_, 1, P)
        assert it == P
        assert np.abs(x - x_ref).max() < 1e-8 * np.abs(x_ref).max(), P
    x_exact = np.linalg.solve(A, s["rhs"])
    assert np.abs(x - x_exact).max() > 1e-4 * np.abs(x_exact).max()   # P = 10 is not converged


def test_mirror_register_trajectory_c1():
    """O3 in MIRROR mode (G = 5, P = 10, the bench's GN shape) against a numpy loop: oracle
    assembly, textbook PCG, Exp(dtheta) R_j / t_j + dt_j (R-A18) -- same energies, same state."""
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    prm = O.params(gn_iters=5, pcg_iters=10, solve_mode=1)
    Rt = O.identity_state(m)
    Es = []
    for _ in range(prm.gn_iters):
        s = O.system(prm, pb, fr, Rt)
        Es.append(s["energy"][4])
        Hd = O.dense_H(s, m)
        x = _textbook_pcg(Hd + prm.lambda_ * np.eye(6 * m), s["rhs"], _block_jacobi(Hd, m, prm.lambda_), 10)
        for j in range(m):
            Rt[j, :9] = (O.exp_so3(x[6 * j:6 * j + 3]) @ Rt[j, :9].reshape(3, 3)).ravel()
            Rt[j, 9:] += x[6 * j + 3:6 * j + 6]
    Es.append(O.system(prm, pb, fr, Rt)["energy"][4])
    Ro, Eo, _ = O.register(prm, pb, fr)
    assert np.abs(Ro - Rt).max() < 1e-9
    assert np.allclose(Eo[:, 4], Es, rtol=1e-10)


def test_oracle_threads_same_result():
    """or_set_threads (bench.py's all-cores column) changes only the summation order."""
    sc, pb, fr, _ = scene_problem("c2")
    m = pb.g.shape[0]
    prm = O.params()
    Rt = random_state(m, np.random.default_rng(4), 0.01, 0.3)
    s1 = O.system(prm, pb, fr, Rt)
    try:
        O.set_threads(4)
        s4 = O.system(prm, pb, fr, Rt)
        o4 = O.fuse(prm, pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], fr, sc["rgb_obs"], 2, pb.g)
    finally:
        O.set_threads(1)
    o1 = O.fuse(prm, pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], fr, sc["rgb_obs"], 2, pb.g)
    H1, H4 = O.dense_H(s1, m), O.dense_H(s4, m)
    assert np.abs(H1 - H4).max() <= 1e-12 * np.abs(H1).max()
    assert np.allclose(s1["energy"], s4["energy"], rtol=1e-12) and s1["n_assoc"] == s4["n_assoc"]
    for key in ("xyz", "nrm", "weight", "stamp", "owner", "lift_idx", "why"):
        np.testing.assert_array_equal(o1[key], o4[key])


# ------------------------------------------------------------------ O8: Alg. 2 Step 5 node regeneration (A36)
def test_regen_spec_cube_and_clusters():
    gr = GOLD["node_regen"]
    lo, e = np.array(gr["cube_corner_min"]), gr["cube_edge"]
    corners = np.array([[lo[0] + e * (i & 1), lo[1] + e * ((i >> 1) & 1), lo[2] + e * (i >> 2)] for i in range(8)])
    g, nbr, _ = O.regenerate_nodes(corners, gr["cube_grid"], 4)
    assert g.shape == (1, 3) and np.allclose(g[0], gr["cube_centroid"], atol=1e-12)
    assert (nbr == -1).all()                                    # no other node
    rng = np.random.default_rng(2)
    pts = np.concatenate([c + rng.uniform(-2, 2, (20, 3)) for c in gr["clusters"]])
    g, nbr, _ = O.regenerate_nodes(pts, gr["cluster_grid"], 1)
    assert g.shape == (2, 3) and nbr[0, 0] == 1 and nbr[1, 0] == 0
    assert np.allclose(g, [pts[:20].astype(np.float32).astype(np.float64).mean(0),
                           pts[20:].astype(np.float32).astype(np.float64).mean(0)], atol=1e-12)
    g4, nbr4, _ = O.regenerate_nodes(pts, gr["cluster_grid"], 4)
    assert (nbr4[:, 1:] == -1).all() and (nbr4[:, 0] == [1, 0]).all()


@pytest.mark.parametrize("seed", range(3))
def test_regen_uniform_cube_brute_force(seed):
    """node count = occupied cells; centroids = per-cell means; N(j) = the n_nbr nearest by a
    brute-force distance table with (distance, index) ties; ascending (kx, ky, kz) node order."""
    gr = GOLD["node_regen"]
    rng = np.random.default_rng(20 + seed)
    pts = rng.uniform(0, gr["uniform_edge"], (gr["uniform_n"], 3)).astype(np.float32)
    s = np.float32(gr["uniform_grid"])
    g, nbr, mg = O.regenerate_nodes(pts, s, 6)
    cells = np.floor(pts / s).astype(np.int64)                      # fp32 division, as A30
    uc, inv = np.unique(cells, axis=0, return_inverse=True)          # lexicographic = (kx, ky, kz)
    assert g.shape[0] == uc.shape[0]
    cnt = np.bincount(inv)
    mean = np.stack([np.bincount(inv, pts[:, a].astype(np.float64)) / cnt for a in range(3)], -1)
    assert np.abs(g - mean).max() < 1e-12
    D = np.linalg.norm(g[:, None] - g[None], axis=-1)
    np.fill_diagonal(D, np.inf)
    for j in range(g.shape[0]):
        order = np.lexsort((np.arange(g.shape[0]), D[j]))[:6]
        assert (nbr[j] == order).all()
    assert (mg >= 0).all()


# ------------------------------------------------------------------ NEXT-2: joint global pose (Eq. 10, A37-A39)
def _Rz(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]])


def _Ry(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, 0, s], [0, 1.0, 0], [-s, 0, c]])


def _Rx(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[1.0, 0, 0], [0, c, -s], [0, s, c]])


def _scope(yaw, pitch, roll):
    """Textbook ZYX composition O = Rz(yaw) Ry(pitch) Rx(roll) (radians)."""
    return _Rz(yaw) @ _Ry(pitch) @ _Rx(roll)


def _pose_increment(pose, x):
    """A37's increment, written out: R <- R Exp(dphi), T <- T + R dtau."""
    R = pose[:9].reshape(3, 3)
    return np.concatenate([(R @ O.exp_so3(x[:3])).ravel(), pose[9:] + R @ x[3:6]])


def _random_pose(rng, rot_deg=8.0, trans=5.0):
    O_ = _scope(*np.deg2rad(rng.uniform(-rot_deg, rot_deg, 3)))
    return np.concatenate([O_.T.ravel(), rng.normal(0, trans, 3)])


def test_pose_euler_zyx_textbook():
    rng = np.random.default_rng(2001)
    for _ in range(50):
        e = np.array([rng.uniform(-np.pi, np.pi), rng.uniform(-1.5, 1.5), rng.uniform(-np.pi, np.pi)])
        assert np.abs(O.euler_zyx(_scope(*e)) - e).max() < 1e-12
    assert np.abs(O.euler_zyx(_Rz(0.3))).max() - 0.3 < 1e-15


def test_pose_prior_golden():
    for c in GOLD["pose_prior"]["cases"]:
        pri = np.concatenate([_scope(*np.deg2rad(c["prior_R_deg_zyx"])).T.ravel(), c["prior_T"]])
        cur = np.concatenate([_scope(*np.deg2rad(c["cur_R_deg_zyx"])).T.ravel(), c["cur_T"]])
        r, J, fl = O.pose_prior(pri, cur)
        assert fl == 0 and np.abs(r - np.array(c["r"])).max() < 1e-12, (c["what"], r)


def test_pose_prior_jacobian_finite_differences():
    rng = np.random.default_rng(2002)
    h = 1e-6
    for _ in range(20):
        pri, cur = _random_pose(rng), _random_pose(rng)
        r, J, fl = O.pose_prior(pri, cur)
        Jfd = np.zeros((6, 6))
        for c in range(6):
            e = np.zeros(6); e[c] = h
            Jfd[:, c] = (O.pose_prior(pri, _pose_increment(cur, e))[0] - O.pose_prior(pri, _pose_increment(cur, -e))[0]) / (2 * h)
        assert np.abs(J - Jfd).max() < 1e-6 * max(1.0, np.abs(J).max()), np.abs(J - Jfd).max()


def test_pose_prior_gimbal_lock_flag():
    cur = np.concatenate([_scope(0.2, np.pi / 2, 0.1).T.ravel(), np.zeros(3)])
    r, J, fl = O.pose_prior(pose12(), cur)
    assert fl == 1 and np.abs(r[:3]).max() == 0 and np.abs(J[:3]).max() == 0


def _joint_fd(prm, pb, fr, Rt, pose, h=1e-5):
    pix, _, _ = O.associate(prm, pb, fr, Rt)   # frozen at the prior's association (a smooth function)
    fsk = O.feature_skin(pb)[:2]
    r0, J = O.residuals_pose(prm, pb, fr, Rt, pose, pix, fsk)
    m = pb.g.shape[0]
    Jfd = np.zeros_like(J)
    for j in range(m):
        for c in range(6):
            rp, _ = O.residuals_pose(prm, pb, fr, apply_perturbation(Rt, j, c, h), pose, pix, fsk)
            rm, _ = O.residuals_pose(prm, pb, fr, apply_perturbation(Rt, j, c, -h), pose, pix, fsk)
            Jfd[:, 6 * j + c] = (rp - rm) / (2 * h)
    for c in range(6):
        e = np.zeros(6); e[c] = h
        rp, _ = O.residuals_pose(prm, pb, fr, Rt, _pose_increment(pose, e), pix, fsk)
        rm, _ = O.residuals_pose(prm, pb, fr, Rt, _pose_increment(pose, -e), pix, fsk)
        Jfd[:, 6 * m + c] = (rp - rm) / (2 * h)
    return J, Jfd, pix


@pytest.mark.parametrize("seed", range(8))
def test_pose_joint_finite_difference_jacobians_small(seed):
    prm, pb, fr, Rt = _small_problem(seed)
    prm.joint_pose = 1
    prm.w_r, prm.w_p = 3.0, 2.0   # O(1) weights so that every block of J is visible in the max-norm
    pose = _pose_increment(np.array(fr.s.pose[:]), np.random.default_rng(700 + seed).normal(0, [0.003] * 3 + [0.2] * 3))
    J, Jfd, pix = _joint_fd(prm, pb, fr, Rt, pose)
    m = pb.g.shape[0]
    assert (pix >= 0).sum() >= 5
    assert np.abs(J[:, 6 * m:]).max() > 0
    rel = np.abs(J - Jfd).max() / np.abs(J).max()
    assert rel < 1e-4, rel
    relp = np.abs(J[:, 6 * m:] - Jfd[:, 6 * m:]).max() / np.abs(J[:, 6 * m:]).max()
    assert relp < 1e-4, relp


def test_pose_joint_assembly_equals_dense_jtj_c1():
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    rng = np.random.default_rng(2003)
    Rt = random_state(m, rng, 0.01, 0.3)
    prm = O.params(joint_pose=1)
    pose = _pose_increment(np.array(fr.s.pose[:]), rng.normal(0, [0.002] * 3 + [0.1] * 3))
    s = O.system_pose(prm, pb, fr, Rt, pose)
    pix, _, _ = O.associate(prm, pb, fr, Rt)
    # the association of the system is taken at the current pose: freeze the same one
    frc = O.Frame(sc["depth"], sc["intr"], pose)
    pix, _, _ = O.associate(prm, pb, frc, Rt)
    r, J = O.residuals_pose(prm, pb, fr, Rt, pose, pix)
    H = O.dense_H(s, m + 1)
    Hd = J.T @ J
    assert np.abs(H - Hd).max() < 1e-9 * np.abs(Hd).max()
    assert np.abs(s["rhs"] + J.T @ r).max() < 1e-9 * np.abs(J.T @ r).max()
    assert abs(s["energy"][6] - r @ r) < 1e-10 * (r @ r)
    assert s["energy"][4] > 0 and s["energy"][5] > 0
    # the node-node part is the fixed-pose system at the same pose (the pose only adds a row / column)
    s0 = O.system(O.params(), pb, frc, Rt)
    H0 = O.dense_H(s0, m)
    assert np.abs(H[:6 * m, :6 * m] - H0).max() < 1e-10 * np.abs(H0).max()
    assert np.abs(s["rhs"][:6 * m] - s0["rhs"]).max() < 1e-10 * np.abs(s0["rhs"]).max()


def test_pose_joint_gn_step_is_dense_solve_and_increment():
    """One joint GN iteration (EXACT) = numpy solve of (J^T J + lambda I) x = -J^T r on the
    oracle's residual stack, then the node (A18) and pose (A37) increments written out."""
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    prm = O.params(joint_pose=1, gn_iters=1, solve_mode=0)
    Rt0 = O.identity_state(m)
    pose0 = np.array(fr.s.pose[:])
    pix, _, _ = O.associate(prm, pb, fr, Rt0)
    r, J = O.residuals_pose(prm, pb, fr, Rt0, pose0, pix)
    x = np.linalg.solve(J.T @ J + prm.lambda_ * np.eye(6 * (m + 1)), -J.T @ r)
    Rt, pose, E, na = O.register_pose(prm, pb, fr)
    Rd = Rt0.copy()
    for j in range(m):
        Rd[j, :9] = (O.exp_so3(x[6 * j:6 * j + 3]) @ Rt0[j, :9].reshape(3, 3)).ravel()
        Rd[j, 9:] += x[6 * j + 3:6 * j + 6]
    assert np.abs(Rt - Rd).max() < 1e-8
    assert np.abs(pose - _pose_increment(pose0, x[6 * m:])).max() < 1e-9
    assert abs(E[0, 6] - r @ r) < 1e-10 * (r @ r) and E[0, 4] == 0 and E[0, 5] == 0


def test_pose_prior_anchoring_and_energy():
    """with w_r, w_p -> 1e12 the refined pose stays at the prior (1e-6) and the nodes
    match the fixed-pose registration; with the paper's weights the joint GN energy falls,
    ends no higher than the fixed-pose one (6 more unknowns, EXACT solves) and the pose
    moves off the prior (E_r + E_p > 0: the stiff priors hold it within ~1e-7)."""
    sc, pb, fr, _ = scene_problem("c1")
    base = dict(gn_iters=3, solve_mode=0)
    Rt_f, E_f, _ = O.register(O.params(**base), pb, fr)
    Rt_a, pose_a, E_a, _ = O.register_pose(O.params(joint_pose=1, w_r=1e12, w_p=1e12, **base), pb, fr)
    pose0 = np.array(fr.s.pose[:])
    assert np.abs(pose_a - pose0).max() < 1e-6
    assert np.abs(Rt_a - Rt_f).max() < 1e-4
    Rt_j, pose_j, E_j, _ = O.register_pose(O.params(joint_pose=1, **base), pb, fr)
    assert (np.diff(E_j[:, 6]) < 0).all() and E_j[-1, 6] <= E_f[-1, 4] * (1 + 1e-9)
    assert E_j[-1, 4] + E_j[-1, 5] > 0 and 0 < np.abs(pose_j - pose0).max() < 1e-6


def test_pose_joint_lm_accepted_energy_decreasing():
    sc, pb, fr, _ = scene_problem("c1")
    prm = O.params(joint_pose=1, gn_iters=8, solve_mode=1, lm=1, lm_mu0=1e-3)
    Rt, pose, E, na, acc = O.register_pose(prm, pb, fr, with_accepted=True)
    ea = E[acc == 1, 6]
    assert (np.diff(ea) < 0).all(), ea
    Ef = O.system_pose(prm, pb, fr, Rt, pose)["energy"][6]
    assert abs(Ef - ea[-1]) < 1e-9 * ea[0]


# ------------------------------------------------------------------ NEXT-4: affine nodes + E_rot (A41-A45)
def random_affine(m, rng, rot_rad=0.02, shear=0.02, trans_mm=0.3):
    """A_j = rotation x (I + small general matrix), t_j random: a non-orthonormal state."""
    At = np.zeros((m, 12))
    for j in range(m):
        At[j, :9] = (O.exp_so3(rng.normal(0, rot_rad, 3)) @ (np.eye(3) + rng.normal(0, shear, (3, 3)))).ravel()
        At[j, 9:] = rng.normal(0, trans_mm, 3)
    return At


def test_rot_spec_examples_and_jacobian():
    """Rot(I) = 0, Rot(2I) = 27 ((4-1)^2 x 3), Rot(30 deg about z) = 0; E_rot = 0 iff
    orthonormal; the Jacobian against central differences."""
    assert np.abs(O.rot_terms(np.eye(3))[0]).max() == 0
    assert abs((O.rot_terms(2 * np.eye(3))[0] ** 2).sum() - 27.0) < 1e-12
    assert (O.rot_terms(rot([0, 0, 1], 30.0))[0] ** 2).sum() < 1e-24
    rng = np.random.default_rng(4001)
    for _ in range(10):
        A = rng.normal(0, 1, (3, 3))
        r, J = O.rot_terms(A)
        # textbook: the Gram matrix of the columns minus I
        G = A.T @ A - np.eye(3)
        assert np.allclose(r, [G[0, 1], G[0, 2], G[1, 2], G[0, 0], G[1, 1], G[2, 2]], atol=1e-12)
        Jfd = np.zeros((6, 9))
        for e in range(9):
            d = np.zeros(9); d[e] = 1e-6
            Jfd[:, e] = (O.rot_terms(A.ravel() + d)[0] - O.rot_terms(A.ravel() - d)[0]) / 2e-6
        assert np.abs(J - Jfd).max() < 1e-8
        assert (r ** 2).sum() > 0   # a random matrix is not orthonormal


def test_aff_normal_warp_golden_and_tangent_invariant():
    """A = diag(2,1,1), n = (1,0,0) -> (1,0,0); the inverse transpose keeps warped tangents
    orthogonal to warped normals: (A u).(A^-T n) = u.n = 0 for random A."""
    pb = single_node_problem([[0.5, 0.2, 50.0]], [[1, 0, 0]])
    At = O.identity_affine(2)
    At[0, :9] = np.diag([2.0, 1.0, 1.0]).ravel()
    _, nh, _, nt, ok = O.warp_aff(pb, At, pose12())
    assert ok[0] and np.allclose(nt[0], [1, 0, 0], atol=1e-15)
    rng = np.random.default_rng(4002)
    for _ in range(20):
        A = np.eye(3) + rng.normal(0, 0.3, (3, 3))
        n = rng.normal(0, 1, 3); n /= np.linalg.norm(n)
        n = n.astype(np.float32).astype(np.float64)   # what the problem stores
        u = np.cross(n, rng.normal(0, 1, 3))
        pb = single_node_problem([[1.0, 2.0, 3.0]], [n])
        At = O.identity_affine(2)
        At[0, :9] = A.ravel()
        _, nh, _, _, ok = O.warp_aff(pb, At, pose12())
        assert ok[0] and abs((A @ u) @ nh[0]) < 1e-12 * np.linalg.norm(A @ u)


def test_aff_reduces_to_se3_on_rotations():
    """With every A_j a rotation the affine model is the SE(3) model: same warp, association,
    data / point / regulariser / feature energies, and E_rot = 0 (two separate code paths)."""
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    Rt = random_state(m, np.random.default_rng(4003), 0.02, 0.3)
    prm = O.params()
    x1 = O.warp(pb, Rt, np.array(fr.s.pose[:]))
    x2 = O.warp_aff(pb, Rt, np.array(fr.s.pose[:]))
    for a, b in zip(x1[:4], x2[:4]):
        assert np.abs(a - b).max() < 1e-12
    p1, w1, _ = O.associate(prm, pb, fr, Rt)
    p2, w2, _ = O.associate_aff(prm, pb, fr, Rt)
    assert (p1 == p2).all() and (w1 == w2).all()
    e1 = O.system(prm, pb, fr, Rt)["energy"]
    e2 = O.system_aff(prm, pb, fr, Rt)["energy"]
    assert np.allclose(e1[:4], e2[:4], rtol=1e-12, atol=1e-12) and e2[4] < 1e-20


def _aff_fd(prm, pb, fr, At, h=1e-6):
    pix, _, _ = O.associate_aff(prm, pb, fr, At)
    fsk = O.feature_skin(pb)[:2]
    r0, J = O.residuals_aff(prm, pb, fr, At, pix, fsk)
    Jfd = np.zeros_like(J)
    for j in range(pb.g.shape[0]):
        for c in range(12):
            Ap = At.copy(); Ap[j, c] += h
            Am = At.copy(); Am[j, c] -= h
            Jfd[:, 12 * j + c] = (O.residuals_aff(prm, pb, fr, Ap, pix, fsk)[0] -
                                  O.residuals_aff(prm, pb, fr, Am, pix, fsk)[0]) / (2 * h)
    return J, Jfd, pix


@pytest.mark.parametrize("seed", range(10))
def test_aff_finite_difference_jacobians_small(seed):
    prm, pb, fr, _ = _small_problem(seed)
    prm.w_rot = 3.0
    At = random_affine(pb.g.shape[0], np.random.default_rng(4100 + seed))
    J, Jfd, pix = _aff_fd(prm, pb, fr, At)
    assert (pix >= 0).sum() >= 5
    rel = np.abs(J - Jfd).max() / np.abs(J).max()
    assert rel < 1e-6, rel


def test_aff_assembly_equals_dense_jtj_c1():
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    At = random_affine(m, np.random.default_rng(4004))
    prm = O.params()
    s = O.system_aff(prm, pb, fr, At)
    pix, _, _ = O.associate_aff(prm, pb, fr, At)
    r, J = O.residuals_aff(prm, pb, fr, At, pix)
    H = O.dense_H_aff(s, m)
    Hd = J.T @ J
    assert np.abs(H - Hd).max() < 1e-10 * np.abs(Hd).max()
    assert np.abs(s["rhs"] + J.T @ r).max() < 1e-10 * np.abs(J.T @ r).max()
    assert abs(s["energy"][5] - r @ r) < 1e-10 * (r @ r)
    assert s["energy"][4] > 0 and s["n_assoc"] == int((pix >= 0).sum())
    # with the features' rows and E_rot's the system is symmetric PSD
    ev = np.linalg.eigvalsh(0.5 * (H + H.T))
    assert ev.min() > -1e-10 * ev.max()


def test_aff_gn_step_is_dense_solve_and_additive_update():
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    prm = O.params(gn_iters=1, solve_mode=0)
    At0 = random_affine(m, np.random.default_rng(4005))
    pix, _, _ = O.associate_aff(prm, pb, fr, At0)
    r, J = O.residuals_aff(prm, pb, fr, At0, pix)
    x = np.linalg.solve(J.T @ J + prm.lambda_ * np.eye(12 * m), -J.T @ r)
    At, E, na = O.register_aff(prm, pb, fr, At0)
    assert np.abs(At - (At0 + x.reshape(m, 12))).max() < 1e-8
    assert abs(E[0, 5] - r @ r) < 1e-10 * (r @ r)


def test_aff_mirror_pcg_is_textbook_pcg():
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    prm = O.params()
    s = O.system_aff(prm, pb, fr, random_affine(m, np.random.default_rng(4006)))
    Hd = O.dense_H_aff(s, m)
    A = Hd + prm.lambda_ * np.eye(12 * m)
    Minv = np.zeros_like(Hd)
    for j in range(m):
        B = Hd[12 * j:12 * j + 12, 12 * j:12 * j + 12]
        Minv[12 * j:12 * j + 12, 12 * j:12 * j + 12] = np.linalg.inv(B + (prm.lambda_ + 1e-9 * np.trace(B) / 12) *
                                                                     np.eye(12))
    for P in (1, 10):
        x_ref = _textbook_pcg(A, s["rhs"], Minv, P)
        x, it = O.solve_aff(s, m, prm.lambda_, 1, P)
        assert it == P and np.abs(x - x_ref).max() < 1e-8 * np.abs(x_ref).max()
    x, _ = O.solve_aff(s, m, prm.lambda_, 0, 0)
    assert np.abs(A @ x - s["rhs"]).max() < 1e-9 * np.abs(s["rhs"]).max()


def test_aff_rigid_motion_recovered():
    """P2 for the affine model: a noise-free rigid tissue motion (Q, c) is recovered with
    A_j = Q (E_rot = 0 there) and t_j = (Q - I) g_j + c."""
    Q, c = rot([1, -2, 0.5], 1.5), np.array([0.8, -0.5, 0.6])
    pb, fr = _rigid_scene(Q, c)
    prm = O.params(w_pt=0.0, gn_iters=10, solve_mode=0)
    At, E, _ = O.register_aff(prm, pb, fr)
    g = pb.g.astype(np.float64)
    assert np.abs(At[:, :9] - Q.ravel()).max() < 1e-4
    assert np.linalg.norm(At[:, 9:] - (g @ (Q - np.eye(3)).T + c), axis=1).max() < 0.01
    assert E[-1, 5] < 1e-3 * E[0, 5]


def test_aff_warp_model_closed_forms():
    sc, pb, fr, _ = scene_problem("c1")
    m = pb.g.shape[0]
    xyz, nrm, g = O.warp_model_aff(pb, O.identity_affine(m))
    assert np.abs(xyz - pb.xyz).max() < 1e-5 and np.abs(g - pb.g).max() == 0
    At = O.identity_affine(m)
    At[:, 9:] = [1.0, -2.0, 0.5]       # common translation: every point moves by it, nodes advance
    xyz, nrm, g = O.warp_model_aff(pb, At)
    assert np.abs(xyz - (pb.xyz.astype(np.float64) + [1.0, -2.0, 0.5])).max() < 1e-9
    assert np.abs(g - (pb.g.astype(np.float64) + [1.0, -2.0, 0.5])).max() < 1e-12


def test_aff_lm_accepted_energy_decreasing_and_mu0_is_gn():
    """The affine oracle's LM: accepted energies strictly decrease, the returned state is the last
    accepted one; with mu0 = 0 and every trial accepted it is the affine GN."""
    sc, pb, fr, _ = scene_problem("c1")
    prm = O.params(gn_iters=8, solve_mode=1, lm=1, lm_mu0=1e-3)
    At, E, na, acc = O.register_aff(prm, pb, fr, with_accepted=True)
    ea = E[acc == 1, 5]
    assert (np.diff(ea) < 0).all(), ea
    assert abs(O.system_aff(prm, pb, fr, At)["energy"][5] - ea[-1]) < 1e-9 * ea[0]
    g = O.register_aff(O.params(gn_iters=2, solve_mode=1), pb, fr)
    l = O.register_aff(O.params(gn_iters=2, solve_mode=1, lm=1, lm_mu0=0.0), pb, fr, with_accepted=True)
    assert (l[3] == 1).all() and np.array_equal(g[0], l[0])
