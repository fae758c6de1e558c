"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

Gates (BASELINE.json north_star, in mm):
  association pix / why bit-exact outside ties (oracle margin <= 1e-6);
  J^T J / J^T r within relative 1e-4 (Cauchy-Schwarz scaled);
  converged nodes within 0.01 mm / 1e-4 rad (MIRROR mode, same G and P);
  warped / fused points within 0.05 mm.
"""
import numpy as np
import pytest

import oracle as O
from paper_1803_02009_b200 import synth
from tests.common import check_fusion, pose12, random_state, rot, scene_problem, state_f32

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1803_02009_b200.mis")


def make_ctx(sc, pb, **kw):
    c = sc["cfg"]
    kw.pop("n_nbr", None)
    prm = M.mis_default_params(k=pb.k, n_nbr=pb.n_nbr, gn_iters=kw.pop("gn_iters", c.gn_iters),
                               pcg_iters=kw.pop("pcg_iters", c.pcg_iters), **kw)
    ctx = M.Context(prm)
    n = pb.xyz.shape[0]
    M.mis_set_model(ctx.ptr, pb.xyz, pb.nrm, sc.get("rgb"), sc.get("weight"), sc.get("stamp"), None,
                    capacity=n + c.H * c.W)
    M.mis_set_graph(ctx.ptr, pb.g, pb.nbr, pb.idx, np.ascontiguousarray(pb.w, np.float32))
    it = sc["intr"]
    M.mis_set_frame(ctx.ptr, sc["depth"], M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"]),
                    sc["pose"])
    if pb.fsrc.shape[0]:
        M.mis_set_features(ctx.ptr, pb.fsrc, pb.fdst)
    return ctx


def oracle_params(ctx_prm, **kw):
    p = ctx_prm
    d = dict(k=p.k, n_nbr=p.n_nbr, w_data=p.w_data, w_pt=p.w_point, w_reg=p.w_reg, w_corr=p.w_corr,
             eps_d=p.eps_d_mm, eps_n_deg=p.eps_n_deg, tau_z=p.tau_z_mm, delta_deg=p.delta_deg, trunc=p.trunc_mm,
             omega_max=p.omega_max, gn_iters=p.gn_iters, pcg_iters=p.pcg_iters, lambda_=p.lambda_, solve_mode=1)
    d.update(kw)
    return O.params(**d)


def order_of(ctx, k):
    return M.mis_get_model(ctx.ptr, k)["ids"]


STATES = ["identity", "rigid", "random"]


def node_state(kind, g, seed=0):
    m = g.shape[0]
    if kind == "identity":
        return O.identity_state(m)
    if kind == "rigid":
        Q, c = rot([1, -2, 0.5], 1.2), np.array([0.4, -0.3, 0.5])
        Rt = np.zeros((m, 12))
        Rt[:, :9] = Q.ravel()
        Rt[:, 9:] = g.astype(np.float64) @ (Q - np.eye(3)).T + c
        return Rt
    return random_state(m, np.random.default_rng(seed), 0.01, 0.3)


# ------------------------------------------------------------------ K1 / K2
@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_frame_prep_parity(cfg):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb)
    nm = M.mis_dbg_frame(ctx.ptr, sc["cfg"].H, sc["cfg"].W)
    q, N, dv, nv = O.frame_prep(fr)
    assert ((nm[..., 3] > 0) == dv).all()
    gv = np.abs(nm[..., :3]).sum(-1) > 0
    assert (gv == nv).all()
    assert np.abs(nm[nv][:, :3] - N[nv]).max() < 2e-5


@pytest.mark.parametrize("cfg,k", [("c1", 4), ("c2", 4), ("c2", 8)])
def test_skin_parity(cfg, k):
    sc, pb, fr, _ = scene_problem(cfg, k=k)
    ctx = make_ctx(sc, pb)
    rng = np.random.default_rng(3)
    pts = (sc["xyz"][rng.choice(len(sc["xyz"]), 4000)] + rng.normal(0, 1, (4000, 3))).astype(np.float32)
    gi, gw = M.mis_skin(ctx.ptr, pts, k)
    oi, ow, om = O.skin(pts, sc["g"], k)
    order = np.argsort(oi, axis=1)
    oi = np.take_along_axis(oi, order, 1)
    ow = np.take_along_axis(ow, order, 1)
    keep = om > 1e-5
    assert keep.mean() > 0.95
    assert (gi[keep] == oi[keep]).all()
    assert np.abs(gw[keep] - ow[keep]).max() < 2e-5


# ------------------------------------------------------------------ association
@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("state", STATES)
def test_association_parity(cfg, state):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb)
    Rt = state_f32(node_state(state, pb.g))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    pix, why = M.mis_dbg_associate(ctx.ptr, pb.xyz.shape[0])
    ids = order_of(ctx, pb.k)
    prm = oracle_params(ctx.params)
    opix, owhy, omg = O.associate(prm, pb, fr, Rt)
    opix, owhy, omg = opix[ids], owhy[ids], omg[ids]
    keep = omg > 1e-6
    assert keep.mean() > 0.99
    bad = np.flatnonzero(keep & ((pix != opix) | (why != owhy)))
    assert bad.size == 0, (bad[:10], pix[bad[:10]], opix[bad[:10]], why[bad[:10]], owhy[bad[:10]])
    assert (opix >= 0).mean() > 0.5


# ------------------------------------------------------------------ normal equations
def dense_from_bsr(s, m):
    H = np.zeros((6 * m, 6 * m))
    for r in range(m):
        for e in range(s["row_ptr"][r], s["row_ptr"][r + 1]):
            c = s["col"][e]
            H[6 * r:6 * r + 6, 6 * c:6 * c + 6] = s["val"][e]
    return H


def check_system(gs, osys, m, tol=1e-4):
    Hg = dense_from_bsr(gs, m)
    Ho = O.dense_H(osys, m)
    d = np.sqrt(np.maximum(np.diag(Ho), 1e-30))
    scale = np.outer(d, d)
    err = np.abs(Hg - Ho) / scale
    assert err.max() < tol, err.max()
    E = osys["energy"][4]
    bt = np.abs(gs["rhs"] - osys["rhs"]) / np.sqrt(np.diag(Ho) * 2 * E)
    assert bt.max() < tol, bt.max()
    # every term on its own (E_data, E_pt, E_reg, E_corr), relative 1e-4; the 1e-9 mm^2 floor only
    # matters for a term that is exactly zero on the oracle side (e.g. E_reg of a rigid-consistent field)
    assert (np.abs(gs["energy"][:4] - osys["energy"][:4]) <= tol * np.abs(osys["energy"][:4]) + 1e-9).all(), \
        (gs["energy"], osys["energy"])
    # structure: every oracle block present in the GPU pattern, symmetric
    assert np.abs(Hg - Hg.T).max() <= 1e-6 * np.abs(Hg).max()


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("state", STATES)
def test_system_parity(cfg, state):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb)
    Rt = state_f32(node_state(state, pb.g, seed=11))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    m = pb.g.shape[0]
    gs = M.mis_dbg_system(ctx.ptr, m)
    prm = oracle_params(ctx.params)
    osys = O.system(prm, pb, fr, Rt)
    osys["prm"] = prm
    check_system(gs, osys, m)


@pytest.mark.parametrize("w_pt", [0.0, 1.0])
def test_system_parity_k8_point_weight(w_pt):
    sc, pb, fr, _ = scene_problem("c2", k=8)
    ctx = make_ctx(sc, pb, w_point=w_pt, n_nbr=pb.n_nbr)
    Rt = state_f32(node_state("random", pb.g, seed=5))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    m = pb.g.shape[0]
    gs = M.mis_dbg_system(ctx.ptr, m)
    prm = oracle_params(ctx.params)
    osys = O.system(prm, pb, fr, Rt)
    osys["prm"] = prm
    check_system(gs, osys, m)


@pytest.mark.parametrize("k", [5, 6, 7])
def test_system_parity_k5_to_k7(k):
    """Every k > 4 instantiation of the tcgen05 K3b (k3b_umma.cu; the k = 8 one runs above and at C5):
    the system of a random node state within the J^T J gate."""
    sc, pb, fr, _ = scene_problem("c2", k=k)
    ctx = make_ctx(sc, pb, n_nbr=pb.n_nbr)
    Rt = state_f32(node_state("random", pb.g, seed=7 + k))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    m = pb.g.shape[0]
    gs = M.mis_dbg_system(ctx.ptr, m)
    prm = oracle_params(ctx.params)
    osys = O.system(prm, pb, fr, Rt)
    osys["prm"] = prm
    check_system(gs, osys, m)


@pytest.mark.parametrize("switch", ["MIS_K3B_UMMA", "MIS_K3A_CHUNKED"])
def test_k_gt4_alternative_paths(switch):
    """The k > 4 alternatives through the same k > 4 system and registration gates, in a subprocess
    (the switches are read once): MIS_K3B_UMMA=0, the FP32 register-tile K3b instead of the tcgen05
    one; MIS_K3A_CHUNKED=0, the per-point K3a (sparse factor state) feeding the tcgen05 K3b."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **{switch: "0"})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
                        "k8_point_weight or k5_to_k7 or c5_shape"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# ------------------------------------------------------------------ full registration (MIRROR)
def rot_err(Ra, Rb):
    c = np.clip((np.trace(Ra @ Rb.T) - 1) / 2, -1, 1)
    return np.arccos(c)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("solver", ["cluster", "cluster_standard", "grid", "grid_standard"])
def test_register_parity_mirror(cfg, solver):
    sc, pb, fr, _ = scene_problem(cfg)
    flags = M.MIS_F_FINAL_ENERGY | {"cluster": 0, "cluster_standard": M.MIS_F_STANDARD_PCG,
                                    "grid": M.MIS_F_GRID_SOLVER,
                                    "grid_standard": M.MIS_F_GRID_SOLVER | M.MIS_F_STANDARD_PCG}[solver]
    ctx = make_ctx(sc, pb, flags=flags)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert (rep["solver_cluster"] > 0) == (not solver.startswith("grid"))
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    Ro, Eo, nao = O.register(oracle_params(ctx.params), pb, fr)
    terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
    rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
    assert terr.max() < 0.01, terr.max()
    assert rerr.max() < 1e-4, rerr.max()
    assert np.allclose(rep["energy"][:, 4], Eo[:, 4], rtol=1e-3)
    assert np.abs(rep["n_assoc"] - nao).max() <= max(3, 1e-4 * pb.xyz.shape[0])


# ------------------------------------------------------------------ warp + fuse
@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_warp_parity(cfg):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb)
    Rt = state_f32(node_state("random", pb.g, seed=21))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    M.mis_warp(ctx.ptr)
    mod = M.mis_get_model(ctx.ptr, pb.k)
    xo, no, go = O.warp_model(pb, Rt)
    ids = mod["ids"]
    assert np.abs(mod["xyz"] - xo[ids]).max() < 0.05
    assert np.abs(mod["nrm"] - no[ids]).max() < 1e-4
    g = M.mis_get_graph(ctx.ptr, np.zeros((pb.g.shape[0], 3), np.float32))
    assert np.abs(g - go).max() < 1e-4
    Rn = M.mis_get_nodes_f64(ctx.ptr, pb.g.shape[0])
    assert np.abs(Rn - O.identity_state(pb.g.shape[0])).max() == 0


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("posed", [False, True])
def test_fuse_parity(cfg, posed):
    """Fusion registration, Eq. 12-15 and the lift, exact outside ties (common.check_fusion).
    posed: a random world->camera pose and random model weights (Eq. 12-14 with omega != 1,
    back-transform R^T(. - T) under a non-identity pose)."""
    sc, pb, fr, _ = scene_problem(cfg)
    if posed:
        rng = np.random.default_rng(17)
        sc = dict(sc)
        sc["pose"] = pose12(rot(rng.normal(size=3), 2.0), rng.normal(0, 0.8, 3))
        sc["weight"] = rng.integers(1, 10, pb.xyz.shape[0]).astype(np.float32)
        fr = O.Frame(sc["depth"], sc["intr"], sc["pose"])
    ctx = make_ctx(sc, pb)
    n = pb.xyz.shape[0]
    cfgo = sc["cfg"]
    owner, why = M.mis_dbg_fuse_register(ctx.ptr, cfgo.H, cfgo.W, n)
    ids = order_of(ctx, pb.k)
    prm = oracle_params(ctx.params)
    o = O.fuse(prm, pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], fr, sc["rgb_obs"], 7, pb.g)
    n_out, stats = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 7)
    check_fusion(M, ctx, pb.k, o, fr, owner, why, ids, 7, n_out, stats)


@pytest.mark.parametrize("gate_mm", [45.0, 120.0])
def test_fuse_parity_wide_gates(gate_mm):
    """tau_z = trunc beyond 42.9 mm (where a 1e-8 mm fixed-point key would overflow 32 bits):
    the key is |dz| / tz quantised to 32 bits, so the per-pixel winner stays exact."""
    sc, pb, fr, _ = scene_problem("c1")
    ctx = make_ctx(sc, pb, tau_z_mm=gate_mm, trunc_mm=gate_mm)
    n = pb.xyz.shape[0]
    cfgo = sc["cfg"]
    owner, why = M.mis_dbg_fuse_register(ctx.ptr, cfgo.H, cfgo.W, n)
    ids = order_of(ctx, pb.k)
    o = O.fuse(oracle_params(ctx.params), pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], fr, sc["rgb_obs"], 3,
               pb.g)
    n_out, stats = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 3)
    check_fusion(M, ctx, pb.k, o, fr, owner, why, ids, 3, n_out, stats)


def test_device_memory_roundtrip():
    torch = pytest.importorskip("torch")
    sc, pb, fr, _ = scene_problem("c1")
    prm = M.mis_default_params()
    ctx = M.Context(prm)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    M.mis_set_model(ctx.ptr, t(pb.xyz), t(pb.nrm), capacity=pb.xyz.shape[0] + 6000)
    M.mis_set_graph(ctx.ptr, t(pb.g), t(pb.nbr))          # device skinning (Eq. 2 on the GPU)
    it = sc["intr"]
    intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
    rep = M.mis_register(ctx.ptr, t(sc["depth"]), intr, sc["pose"], t(pb.fsrc), t(pb.fdst))
    r = M.report_dict(rep)
    assert r["status"] == 0 and r["energy"][-2, 4] < r["energy"][0, 4]
    out = torch.zeros((pb.g.shape[0], 12), dtype=torch.float32, device="cuda")
    M.mis_get_nodes(ctx.ptr, out)
    assert torch.isfinite(out).all()


def test_sequence_runs_and_grows():
    cfgo = synth.CONFIGS["c1"]
    base, frames = synth.make_sequence_frames("c1", 4)
    prm = M.mis_default_params()
    ctx = M.Context(prm)
    n0 = base["xyz"].shape[0]
    M.mis_set_model(ctx.ptr, base["xyz"], base["nrm"], base["rgb"], base["weight"], base["stamp"], capacity=200_000)
    M.mis_set_graph(ctx.ptr, base["g"], base["nbr"])
    it = base["intr"]
    intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
    n = n0
    for f in frames:
        rep = M.report_dict(M.mis_register(ctx.ptr, f["depth"], intr, f["pose"], f["feat_src"], f["feat_dst"]))
        assert rep["status"] == 0
        M.mis_warp(ctx.ptr)
        n2, st = M.mis_fuse(ctx.ptr, f["rgb_obs"], f["frame"])
        assert n2 == n + st[1] and st[0] + st[1] == st[2]
        n = n2
    mod = M.mis_get_model(ctx.ptr, 4)
    assert np.isfinite(mod["xyz"]).all() and len(np.unique(mod["ids"])) == n


def test_empty_model_and_errors():
    sc, pb, fr, _ = scene_problem("c1")
    ctx = M.Context(M.mis_default_params())
    with pytest.raises(M.MisError):
        M.mis_register(ctx.ptr)                       # no model / graph: MIS_E_STATE
    M.mis_set_model(ctx.ptr, np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32), capacity=10)
    M.mis_set_graph(ctx.ptr, pb.g, pb.nbr)
    it = sc["intr"]
    intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
    rep = M.report_dict(M.mis_register(ctx.ptr, sc["depth"], intr, sc["pose"]))
    assert rep["n_assoc"][0] == 0
    bad = pb.nbr.copy()
    bad[0, 0] = 0                                    # self edge
    with pytest.raises(M.MisError):
        M.mis_set_graph(ctx.ptr, pb.g, bad)
    with pytest.raises(M.MisError):
        M.mis_set_frame(ctx.ptr, sc["depth"], M.intrinsics(-1, 1, 1, 1, it["W"], it["H"]), sc["pose"])


def test_device_graph_validation_deferred():
    """Device-memory mis_set_graph does not synchronise: bad ids surface at the next register."""
    torch = pytest.importorskip("torch")
    sc, pb, fr, _ = scene_problem("c1")
    ctx = M.Context(M.mis_default_params())
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    M.mis_set_model(ctx.ptr, t(pb.xyz), t(pb.nrm), capacity=pb.xyz.shape[0] + 6000)
    bad = pb.nbr.copy()
    bad[3, 1] = pb.g.shape[0] + 7                     # out of range
    M.mis_set_graph(ctx.ptr, t(pb.g), t(bad))          # returns without a host sync
    it = sc["intr"]
    intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
    with pytest.raises(M.MisError, match="neighbour list"):
        M.mis_register(ctx.ptr, t(sc["depth"]), intr, sc["pose"])
    with pytest.raises(M.MisError):                    # the graph is unbound afterwards
        M.mis_register(ctx.ptr)
    M.mis_set_graph(ctx.ptr, t(pb.g), t(pb.nbr))        # a valid graph binds again
    r = M.report_dict(M.mis_register(ctx.ptr, t(sc["depth"]), intr, sc["pose"]))
    assert r["status"] == 0


# ------------------------------------------------------------------ C5-shaped registration at C2 size
@pytest.mark.parametrize("solver", ["grid", "cluster"])
def test_register_parity_c5_shape(solver):
    """C5's method shape (k = 8, n_nbr = 8, G = 8, P = 20; BASELINE configs[4]) on the C2 scene,
    against the oracle's MIRROR registration (same G and P): the grid-wide PCG is C5's solver."""
    sc = synth.make_scene("c2", 1)
    k = 8
    nbr = synth.node_graph(sc["g"], 8)
    idx, w, _ = O.skin(sc["xyz"], sc["g"], k)
    _, _, fm = O.skin(sc["feat_src"], sc["g"], k)
    keep = fm > 1e-4
    pb = O.Problem(sc["xyz"], sc["nrm"], idx, w.astype(np.float32), sc["g"], nbr, sc["feat_src"][keep],
                   sc["feat_dst"][keep])
    fr = O.Frame(sc["depth"], sc["intr"], sc["pose"])
    flags = M.MIS_F_FINAL_ENERGY | (M.MIS_F_GRID_SOLVER if solver == "grid" else 0)
    ctx = make_ctx(sc, pb, gn_iters=8, pcg_iters=20, flags=flags)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert rep["status"] == 0
    assert (rep["solver_cluster"] > 0) == (solver == "cluster")
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    Ro, Eo, nao = O.register(oracle_params(ctx.params), pb, fr)
    terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
    rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
    assert terr.max() < 0.01, terr.max()
    assert rerr.max() < 1e-4, rerr.max()
    assert np.allclose(rep["energy"][:, 4], Eo[:, 4], rtol=1e-3)
    assert np.abs(rep["n_assoc"] - nao).max() <= max(3, 1e-4 * pb.xyz.shape[0])


# ------------------------------------------------------------------ error paths (mis.h)
@pytest.mark.parametrize("solver", ["cluster", "grid"])
def test_numeric_failure_rolls_back(solver):
    """MIS_E_NUMERIC: a non-finite GN step (here: a NaN feature observation makes b non-finite)
    rolls the node state back to before the failing iteration -- the identity, since it is the
    first -- and the context stays usable: the next registration matches the oracle."""
    sc, pb, fr, _ = scene_problem("c1")
    flags = M.MIS_F_GRID_SOLVER if solver == "grid" else 0
    ctx = make_ctx(sc, pb, flags=flags)
    bad = pb.fdst.copy()
    bad[0, 1] = np.nan
    with pytest.raises(M.MisError) as e:
        M.mis_register(ctx.ptr, None, None, None, pb.fsrc, bad)
    assert e.value.status == 7
    m = pb.g.shape[0]
    assert (M.mis_get_nodes_f64(ctx.ptr, m) == O.identity_state(m)).all()
    rep = M.report_dict(M.mis_register(ctx.ptr, None, None, None, pb.fsrc, pb.fdst))
    assert rep["status"] == 0
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    Ro, _, _ = O.register(oracle_params(ctx.params), pb, fr)
    assert np.abs(Rg[:, 9:] - Ro[:, 9:]).max() < 0.01 and np.abs(Rg[:, :9] - Ro[:, :9]).max() < 1e-4


def test_capacity_exceeded_leaves_model_unchanged():
    """MIS_E_CAPACITY: the frame's lift would exceed the capacity -> neither the Eq. 12-15 update
    of the registered points nor any lifted point is applied, the size and ids are unchanged, and
    a later fusion with room proceeds normally (no id consumed)."""
    sc, pb, fr, _ = scene_problem("c1")
    c = sc["cfg"]
    prm = M.mis_default_params(k=pb.k, n_nbr=pb.n_nbr)
    ctx = M.Context(prm)
    n = pb.xyz.shape[0]
    M.mis_set_model(ctx.ptr, pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], None, capacity=n + 10)
    M.mis_set_graph(ctx.ptr, pb.g, pb.nbr, pb.idx, np.ascontiguousarray(pb.w, np.float32))
    it = sc["intr"]
    M.mis_set_frame(ctx.ptr, sc["depth"], M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"]),
                    sc["pose"])
    before = M.mis_get_model(ctx.ptr, pb.k)
    with pytest.raises(M.MisError) as e:
        M.mis_fuse(ctx.ptr, sc["rgb_obs"], 5)
    assert e.value.status == 6
    after = M.mis_get_model(ctx.ptr, pb.k)
    for key in before:
        np.testing.assert_array_equal(after[key], before[key])
    # same model into a context with room: the lifted ids start at n (nothing was consumed)
    M.mis_set_model(ctx.ptr, pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], None, capacity=n + c.H * c.W)
    M.mis_set_graph(ctx.ptr, pb.g, pb.nbr, pb.idx, np.ascontiguousarray(pb.w, np.float32))
    n_out, st = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 5)
    ids = M.mis_get_model(ctx.ptr, pb.k)["ids"]
    assert n_out == n + st[1] and np.array_equal(np.sort(ids), np.arange(n_out))


def test_workspace_binding():
    """§8(b) mis_workspace_bytes / mis_bind_workspace: a torch allocation backs every buffer of a
    full frame (register, warp, fuse, filter) -- no device memory is taken outside it -- with the
    same result as a cudaMalloc'ed context; order and size errors are reported."""
    torch = pytest.importorskip("torch")
    sc, pb, fr, _ = scene_problem("c2")
    c = sc["cfg"]
    n, m = pb.xyz.shape[0], pb.g.shape[0]
    cap = n + 2 * c.H * c.W
    it = sc["intr"]
    intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])

    def frame(ctx):
        M.mis_set_model(ctx.ptr, pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], None, capacity=cap)
        M.mis_set_graph(ctx.ptr, pb.g, pb.nbr)
        rep = M.report_dict(M.mis_register(ctx.ptr, sc["depth"], intr, sc["pose"], pb.fsrc, pb.fdst))
        nodes = M.mis_get_nodes_f64(ctx.ptr, m)
        M.mis_warp(ctx.ptr)
        n1, _ = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 1)
        n2, _ = M.mis_filter(ctx.ptr, 0.5, 1, 10, 3.0)
        return rep, nodes, n1, n2

    ref = frame(M.Context(M.mis_default_params()))
    ctx = M.Context(M.mis_default_params())
    nb = M.mis_workspace_bytes(ctx.ptr, cap, m, c.H, c.W)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    M.mis_bind_workspace(ctx.ptr, ws)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    got = frame(ctx)
    torch.cuda.synchronize()
    assert free0 - torch.cuda.mem_get_info()[0] < 4 << 20      # nothing (beyond driver noise) outside the workspace
    assert got[0]["status"] == 0 and np.abs(got[1] - ref[1]).max() < 1e-3   # fp32 atomic order only
    assert abs(got[2] - ref[2]) <= 10 and abs(got[3] - ref[3]) <= 10
    with pytest.raises(M.MisError) as e:
        M.mis_bind_workspace(ctx.ptr, ws)                      # already bound
    assert e.value.status == 2
    small = M.Context(M.mis_default_params())
    tiny = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    M.mis_bind_workspace(small.ptr, tiny)
    with pytest.raises(M.MisError) as e:
        M.mis_set_model(small.ptr, pb.xyz, pb.nrm, capacity=cap)
    assert e.value.status == 5                                 # MIS_E_NOMEM, names the size
    late = M.Context(M.mis_default_params())
    M.mis_set_model(late.ptr, pb.xyz, pb.nrm, capacity=cap)
    with pytest.raises(M.MisError) as e:
        M.mis_bind_workspace(late.ptr, ws)
    assert e.value.status == 2
