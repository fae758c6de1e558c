"""GPU parity at BASELINE.json's full sizes (configs[2..4]) -- the sizes bench.py times.

c3 (the bench workload, 640x480, 300k points, ~1000 nodes): every stage element by
element against the fp64 oracle on the whole problem, in the launch configuration
bench.py uses (default parameters, device skinning, cluster-resident pipelined PCG).
c4 (2M points, ~4000 nodes, 1280x1024): whole-problem association and normal
equations (block-by-block, sparse), and MIRROR registration on the solver the
library picks at that size (the grid-cooperative PCG: the system does not fit one
16-CTA cluster).
c5 (10M points, ~16k nodes, k=8): the device skinning and association on a seeded
sample of 20k points one by one (a point's association depends only on its own
inputs), properties that hold at any size (monotone energy, finite state, symmetric
system), and -- with the oracle on every host core (~75 s on the GPU box) -- the
whole-problem normal equations block by block and the MIRROR registration.

Gates as in test_gpu_parity.py.
"""
import numpy as np
import pytest

import oracle as O
from paper_1803_02009_b200 import synth
from tests.common import check_fusion, scene_problem, state_f32
from tests.test_gpu_lm import _check_lm
from tests.test_gpu_parity import make_ctx, node_state, oracle_params, order_of, rot_err

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1803_02009_b200.mis")

_CACHE = {}


def problem(cfg):
    if cfg not in _CACHE:
        _CACHE[cfg] = scene_problem(cfg)
    return _CACHE[cfg]


def check_system_sparse(gs, osys, m, tol=1e-4):
    """J^T J blocks compared block by block (no dense 6m x 6m matrix), Cauchy-Schwarz scaled."""
    rp, col, val = gs["row_ptr"], gs["col"], gs["val"].astype(np.float64)
    grow = np.repeat(np.arange(m), np.diff(rp))
    gkey = grow.astype(np.int64) * m + col
    assert (np.diff(gkey) > 0).all()                     # CSR rows sorted, no duplicates
    # oracle blocks, both triangles
    ob = {}
    for r, c, B in zip(osys["rows"], osys["cols"], osys["vals"]):
        ob[(r, c)] = ob.get((r, c), 0) + B
        if r != c:
            ob[(c, r)] = ob.get((c, r), 0) + B.T
    dg = np.zeros((m, 6))
    for j in range(m):
        if (j, j) in ob:
            dg[j] = np.sqrt(np.maximum(np.diag(ob[(j, j)]), 1e-30))
        else:
            dg[j] = 1e-15
    okeys = np.array(sorted(r * m + c for (r, c) in ob), np.int64)
    missing = np.setdiff1d(okeys, gkey)
    assert missing.size == 0, missing[:10]               # every oracle block is in the GPU pattern
    worst = 0.0
    for e in range(gkey.size):
        r, c = int(grow[e]), int(col[e])
        Bo = ob.get((r, c), np.zeros((6, 6)))
        err = np.abs(val[e] - Bo) / np.outer(dg[r], dg[c])
        worst = max(worst, float(err.max()))
    assert worst < tol, worst
    # symmetry of the stored pattern
    pos = {int(k): i for i, k in enumerate(gkey)}
    for e in range(0, gkey.size, 7):
        r, c = int(grow[e]), int(col[e])
        assert np.abs(val[e] - val[pos[c * m + r]].T).max() <= 1e-6 * np.abs(val[e]).max() + 1e-30
    E = osys["energy"][4]
    bt = np.abs(gs["rhs"] - osys["rhs"]) / np.sqrt(dg.ravel() ** 2 * 2 * E)
    assert bt.max() < tol, bt.max()
    # every energy term on its own, relative 1e-4 (test_gpu_parity.check_system)
    assert (np.abs(gs["energy"][:4] - osys["energy"][:4]) <= tol * np.abs(osys["energy"][:4]) + 1e-9).all(), \
        (gs["energy"], osys["energy"])


# ------------------------------------------------------------------ c3: the bench workload, whole problem
def test_c3_device_skinning_full():
    sc, pb, fr, margin = problem("c3")
    c = sc["cfg"]
    ctx = M.Context(M.mis_default_params(k=c.k, n_nbr=c.n_nbr, gn_iters=c.gn_iters, pcg_iters=c.pcg_iters))
    n = pb.xyz.shape[0]
    M.mis_set_model(ctx.ptr, pb.xyz, pb.nrm, capacity=n + c.H * c.W)
    M.mis_set_graph(ctx.ptr, pb.g, pb.nbr)               # device skinning, as bench.py does
    mod = M.mis_get_model(ctx.ptr, c.k)
    ids = mod["ids"]
    oi = np.sort(pb.idx, axis=1)[ids]
    keep = margin[ids] > 1e-5
    assert keep.mean() > 0.99
    assert (mod["knn_idx"][keep] == oi[keep]).all()


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_association_full(cfg):
    sc, pb, fr, _ = problem(cfg)
    ctx = make_ctx(sc, pb)
    Rt = state_f32(node_state("random", pb.g, seed=31))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    pix, why = M.mis_dbg_associate(ctx.ptr, pb.xyz.shape[0])
    ids = order_of(ctx, pb.k)
    opix, owhy, omg = O.associate(oracle_params(ctx.params), pb, fr, Rt)
    opix, owhy, omg = opix[ids], owhy[ids], omg[ids]
    keep = omg > 1e-6
    assert keep.mean() > 0.99
    bad = np.flatnonzero(keep & ((pix != opix) | (why != owhy)))
    assert bad.size == 0, (bad.size, bad[:10], pix[bad[:10]], opix[bad[:10]])
    assert (opix >= 0).mean() > 0.5


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_system_full(cfg):
    sc, pb, fr, _ = problem(cfg)
    ctx = make_ctx(sc, pb)
    Rt = state_f32(node_state("random", pb.g, seed=37))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    m = pb.g.shape[0]
    gs = M.mis_dbg_system(ctx.ptr, m)
    prm = oracle_params(ctx.params)
    osys = O.system(prm, pb, fr, Rt)
    osys["prm"] = prm
    check_system_sparse(gs, osys, m)


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_register_full_mirror(cfg):
    """Whole registration (G x P fixed) in the launch configuration bench.py uses."""
    sc, pb, fr, _ = problem(cfg)
    ctx = make_ctx(sc, pb, flags=M.MIS_F_FINAL_ENERGY)
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert rep["status"] == 0
    assert (rep["solver_cluster"] > 0) == (cfg == "c3")   # c3 fits one 16-CTA cluster, c4 does not
    m = pb.g.shape[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    Ro, Eo, nao = O.register(oracle_params(ctx.params), pb, fr)
    terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
    rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
    assert terr.max() < 0.01, terr.max()                   # 1e-5 m
    assert rerr.max() < 1e-4, rerr.max()
    assert np.allclose(rep["energy"][:, 4], Eo[:, 4], rtol=1e-3)
    assert np.abs(rep["n_assoc"] - nao).max() <= max(3, 1e-4 * pb.xyz.shape[0])


def test_c3_warp_and_fuse_full():
    sc, pb, fr, _ = problem("c3")
    ctx = make_ctx(sc, pb)
    n = pb.xyz.shape[0]
    c = sc["cfg"]
    owner, why = M.mis_dbg_fuse_register(ctx.ptr, c.H, c.W, n)
    ids = order_of(ctx, pb.k)
    o = O.fuse(oracle_params(ctx.params), pb.xyz, pb.nrm, sc["rgb"], sc["weight"], sc["stamp"], fr,
               sc["rgb_obs"], 9, pb.g)
    n_out, stats = M.mis_fuse(ctx.ptr, sc["rgb_obs"], 9)
    check_fusion(M, ctx, pb.k, o, fr, owner, why, ids, 9, n_out, stats)
    # warp with a random field on a fresh context
    ctx = make_ctx(sc, pb)
    Rt = state_f32(node_state("random", pb.g, seed=41))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    M.mis_warp(ctx.ptr)
    mod = M.mis_get_model(ctx.ptr, pb.k)
    xo, no, _ = O.warp_model(pb, Rt)
    assert np.abs(mod["xyz"] - xo[mod["ids"]]).max() < 0.05
    assert np.abs(mod["nrm"] - no[mod["ids"]]).max() < 1e-4


# ------------------------------------------------------------------ c5: sampled outputs + properties
@pytest.fixture(scope="module")
def c5():
    sc = synth.make_scene("c5", 1)
    c = sc["cfg"]
    ctx = M.Context(M.mis_default_params(k=c.k, n_nbr=c.n_nbr, gn_iters=c.gn_iters, pcg_iters=c.pcg_iters,
                                         flags=M.MIS_F_FINAL_ENERGY))
    n = sc["xyz"].shape[0]
    M.mis_set_model(ctx.ptr, sc["xyz"], sc["nrm"], capacity=n + c.H * c.W)
    M.mis_set_graph(ctx.ptr, sc["g"], sc["nbr"])            # device skinning of all 10M points
    it = sc["intr"]
    M.mis_set_frame(ctx.ptr, sc["depth"], M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"]),
                    sc["pose"])
    M.mis_set_features(ctx.ptr, sc["feat_src"], sc["feat_dst"])
    rng = np.random.default_rng(55)
    sample = np.sort(rng.choice(n, 20_000, replace=False))
    return sc, ctx, sample


def test_c5_sampled_skinning_and_association(c5):
    sc, ctx, sample = c5
    c = sc["cfg"]
    n = sc["xyz"].shape[0]
    mod = M.mis_get_model(ctx.ptr, c.k)
    inv = np.empty(n, np.int64)
    inv[mod["ids"]] = np.arange(n)
    oi, ow, om = O.skin(sc["xyz"][sample], sc["g"], c.k)
    order = np.argsort(oi, axis=1)
    oi, ow = np.take_along_axis(oi, order, 1), np.take_along_axis(ow, order, 1)
    gpos = inv[sample]
    keep = om > 1e-5
    assert keep.mean() > 0.99
    assert (mod["knn_idx"][gpos][keep] == oi[keep]).all()
    assert np.abs(mod["knn_w"][gpos][keep] - ow[keep]).max() < 2e-5
    # association of the sampled points under a random field: the oracle sees only the sample
    Rt = state_f32(node_state("random", sc["g"], seed=57))
    M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
    pix, why = M.mis_dbg_associate(ctx.ptr, n)
    pb = O.Problem(sc["xyz"][sample], sc["nrm"][sample], oi, ow.astype(np.float32), sc["g"], sc["nbr"])
    fr = O.Frame(sc["depth"], sc["intr"], sc["pose"])
    opix, owhy, omg = O.associate(oracle_params(ctx.params), pb, fr, Rt)
    ok = keep & (omg > 1e-6)
    assert ok.mean() > 0.98
    assert (pix[gpos][ok] == opix[ok]).all() and (why[gpos][ok] == owhy[ok]).all()
    assert (opix >= 0).mean() > 0.3


def test_c5_register_properties(c5):
    sc, ctx, _ = c5
    m = sc["g"].shape[0]
    M.mis_dbg_set_nodes(ctx.ptr, O.identity_state(m).astype(np.float32))
    gs = M.mis_dbg_system(ctx.ptr, m)
    rp, col, val = gs["row_ptr"], gs["col"], gs["val"]
    grow = np.repeat(np.arange(m), np.diff(rp))
    diag = np.array([val[rp[j] + np.searchsorted(col[rp[j]:rp[j + 1]], j)] for j in range(m)])
    assert (np.einsum("jii->ji", diag) >= 0).all()
    key = grow.astype(np.int64) * m + col
    pos = np.searchsorted(key, col.astype(np.int64) * m + grow)
    assert (key[pos] == col.astype(np.int64) * m + grow).all()
    sym = np.abs(val - val[pos].transpose(0, 2, 1)).max()
    assert sym <= 1e-6 * np.abs(val).max()
    rep = M.report_dict(M.mis_register(ctx.ptr))
    assert rep["status"] == 0
    E = rep["energy"][:, 4]
    G = sc["cfg"].gn_iters
    assert np.isfinite(E[:G + 1]).all() and E[G] < E[0]
    Rg = M.mis_get_nodes_f64(ctx.ptr, m)
    assert np.isfinite(Rg).all()
    R = Rg[:, :9].reshape(-1, 3, 3)
    assert np.abs(R @ R.transpose(0, 2, 1) - np.eye(3)).max() < 1e-6     # SE(3) state stays on the manifold


# ------------------------------------------------------------------ c5: the whole problem on all host cores
def test_c5_system_and_register_full():
    """BASELINE's largest config (10M points, k = 8: the tcgen05 K3b, chunked sparse K3a, grid PCG) against
    the oracle on the WHOLE problem: the oracle skins all 10M points and assembles / registers in fp64 on
    every host core (or_set_threads changes only its summation order, tests/test_oracle_pins.py).  The
    normal equations block by block under a random field (gates of test_system_full), then the MIRROR
    registration in bench.py's launch configuration (gates of test_register_full_mirror)."""
    import os
    O.set_threads(os.cpu_count() or 1)
    try:
        sc, pb, fr, _ = problem("c5")
        ctx = make_ctx(sc, pb)
        m = pb.g.shape[0]
        Rt = state_f32(node_state("random", pb.g, seed=61))
        M.mis_dbg_set_nodes(ctx.ptr, Rt.astype(np.float32))
        gs = M.mis_dbg_system(ctx.ptr, m)
        prm = oracle_params(ctx.params)
        osys = O.system(prm, pb, fr, Rt)
        osys["prm"] = prm
        check_system_sparse(gs, osys, m)
        del gs, osys
        ctx = make_ctx(sc, pb, flags=M.MIS_F_FINAL_ENERGY)
        rep = M.report_dict(M.mis_register(ctx.ptr))
        assert rep["status"] == 0
        Rg = M.mis_get_nodes_f64(ctx.ptr, m)
        Ro, Eo, nao = O.register(oracle_params(ctx.params), pb, fr)
    finally:
        O.set_threads(1)
    terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
    rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
    assert terr.max() < 0.01, terr.max()                   # 1e-5 m
    assert rerr.max() < 1e-4, rerr.max()
    assert np.allclose(rep["energy"][:, 4], Eo[:, 4], rtol=1e-3)
    assert np.abs(rep["n_assoc"] - nao).max() <= max(3, 1e-4 * pb.xyz.shape[0])


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_lm_full(cfg):
    """MIS_F_LM in bench.py's `lm` leg configuration at C4 and C5 (the grid PCG carries the accept /
    reject decisions; C5 with the tcgen05 K3b) against the oracle's LM on every host core: decisions up
    to the first near tie, trial energies, and the nodes when no tie occurs (test_gpu_lm.py gates)."""
    import os
    O.set_threads(os.cpu_count() or 1)
    try:
        sc, pb, fr, _ = problem(cfg)
        G = sc["cfg"].gn_iters
        ctx = make_ctx(sc, pb, flags=M.MIS_F_LM)
        rep = M.report_dict(M.mis_register(ctx.ptr))
        assert rep["status"] == 0 and rep["solver_cluster"] == 0
        m = pb.g.shape[0]
        Rg = M.mis_get_nodes_f64(ctx.ptr, m)
        Ro, Eo, _, acco = O.register(oracle_params(ctx.params, lm=1, lm_mu0=1e-3, gn_iters=G), pb, fr,
                                     with_accepted=True)
    finally:
        O.set_threads(1)
    ties = _check_lm(rep, Eo, acco, G)
    if not ties:
        terr = np.linalg.norm(Rg[:, 9:] - Ro[:, 9:], axis=1)
        rerr = np.array([rot_err(Rg[j, :9].reshape(3, 3), Ro[j, :9].reshape(3, 3)) for j in range(m)])
        assert terr.max() < 0.01 and rerr.max() < 1e-4, (terr.max(), rerr.max())
