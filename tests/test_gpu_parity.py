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
from tests.common import pose12, random_state, rot, scene_problem, state_f32

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
    p_ = osys["prm"]
    w = np.array([p_.w_data, p_.w_pt, p_.w_reg, p_.w_corr])
    assert (np.abs(gs["energy"][:4] - osys["energy"][:4]) * w <= tol * E + 1e-12).all(), (gs["energy"], osys["energy"])
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


# ------------------------------------------------------------------ full registration (MIRROR)
def rot_err(Ra, Rb):
    c = np.clip((np.trace(Ra @ Rb.T) - 1) / 2, -1, 1)
    return np.arccos(c)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("solver", ["cluster", "cluster_standard", "grid"])
def test_register_parity_mirror(cfg, solver):
    sc, pb, fr, _ = scene_problem(cfg)
    flags = M.MIS_F_FINAL_ENERGY | {"cluster": 0, "cluster_standard": M.MIS_F_STANDARD_PCG,
                                    "grid": M.MIS_F_GRID_SOLVER}[solver]
    ctx = make_ctx(sc, pb, flags=flags)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert (rep["solver_cluster"] > 0) == (solver != "grid")
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
def test_fuse_parity(cfg):
    sc, pb, fr, _ = scene_problem(cfg)
    ctx = make_ctx(sc, pb)
    n = pb.xyz.shape[0]
    cfgo = sc["cfg"]
    owner, why = M.mis_dbg_fuse_register(ctx.ptr, cfgo.H, cfgo.W, n)
    ids = order_of(ctx, pb.k)
    prm = oracle_params(ctx.params)
    o = O.fuse(prm, pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], fr, sc["rgb_obs"], 7, pb.g)
    # owner: GPU internal index -> caller id
    gown = np.where(owner >= 0, ids[np.maximum(owner, 0)], -1)
    gate_ok = np.ones(n, bool)
    gate_ok[ids] = True
    tie = o["key_margin"] <= 1e-6
    # pixels whose candidate points all have clear gate decisions
    assert ((gown == o["owner"]) | tie).mean() > 0.999
    bad = np.flatnonzero((gown != o["owner"]) & ~tie)
    near = o["gate_margin"][o["owner"][bad][o["owner"][bad] >= 0]] if bad.size else np.zeros(0)
    assert bad.size == 0 or (near <= 1e-6).all(), bad[:10]
    assert (why == o["why"][ids]).mean() > 0.999
    # apply
    n_out, stats = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 7)
    assert n_out == n + o["n_lift"]
    assert stats[1] == o["n_lift"]
    mod = M.mis_get_model(ctx.ptr, pb.k)
    gid = mod["ids"]
    old = gid < n
    assert np.abs(mod["xyz"][old] - o["xyz"][gid[old]]).max() < 0.05
    assert (mod["weight"][old] == o["weight"][gid[old]]).mean() > 0.999
    assert (mod["stamp"][old] == o["stamp"][gid[old]]).mean() > 0.999
    assert np.abs(mod["rgb"][old] - o["rgb"][gid[old]]).max() < 1e-3
    # lifted points: ids n.. in row-major pixel order
    new = ~old
    assert np.abs(mod["xyz"][new] - o["xyz"][gid[new]]).max() < 0.05
    assert (mod["weight"][new] == 1).all() and (mod["stamp"][new] == 7).all()
    li = gid[new] - n
    lm = o["lift_margin"][li] > 1e-5
    oi = np.sort(o["lift_idx"][li], axis=1)
    assert (mod["knn_idx"][new][lm] == oi[lm]).all()


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
