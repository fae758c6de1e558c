"""Shared test helpers: build oracle problems from the seeded synthetic scenes."""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_1803_02009_b200 import synth


def rot(axis, deg):
    axis = np.asarray(axis, np.float64)
    return O.exp_so3(axis / np.linalg.norm(axis) * np.deg2rad(deg))


def pose12(R=None, T=None):
    R = np.eye(3) if R is None else np.asarray(R, np.float64)
    T = np.zeros(3) if T is None else np.asarray(T, np.float64)
    return np.concatenate([R.ravel(), T])


def scene_problem(cfg="c1", frame=1, k=None, with_features=True, drop_feature_ties=1e-4, seed_offset=0):
    """Synthetic scene + oracle skinning (Eq. 2) of the model points."""
    sc = synth.make_scene(cfg, frame, seed_offset)
    c = sc["cfg"]
    k = c.k if k is None else k
    idx, w, margin = O.skin(sc["xyz"], sc["g"], k)
    fsrc, fdst = (sc["feat_src"], sc["feat_dst"]) if with_features else (None, None)
    if with_features and drop_feature_ties:
        _, _, fm = O.skin(fsrc, sc["g"], k)
        keep = fm > drop_feature_ties
        fsrc, fdst = fsrc[keep], fdst[keep]
    pb = O.Problem(sc["xyz"], sc["nrm"], idx, w.astype(np.float32), sc["g"], sc["nbr"], fsrc, fdst)
    fr = O.Frame(sc["depth"], sc["intr"], sc["pose"])
    return sc, pb, fr, margin


def random_state(m, rng, rot_rad=0.03, trans_mm=0.5):
    Rt = np.zeros((m, 12))
    for j in range(m):
        Rt[j, :9] = O.exp_so3(rng.normal(0, rot_rad, 3)).ravel()
        Rt[j, 9:] = rng.normal(0, trans_mm, 3)
    return Rt


def apply_perturbation(Rt, j, comp, h):
    """Left perturbation of node j: comp 0-2 rotation (Exp(h e_c) R_j), 3-5 translation."""
    X = Rt.copy()
    if comp < 3:
        e = np.zeros(3)
        e[comp] = h
        X[j, :9] = (O.exp_so3(e) @ X[j, :9].reshape(3, 3)).ravel()
    else:
        X[j, 9 + comp - 3] += h
    return X


def state_f32(Rt):
    """The fp32 node state both sides receive in stage-wise parity (exact upcast)."""
    return np.asarray(Rt, np.float32).astype(np.float64)


def check_fusion(M, ctx, k, o, fr, owner, why, ids, frame_index, n_out, stats, tie=1e-6):
    """Alg. 1 + Eq. 12-15 + Alg. 2 Step 3 parity, exact outside ties.

    owner / why: mis_dbg_fuse_register (GPU internal indices / order) taken before the
    fusion; ids: the caller ids of the internal order then; o: oracle O.fuse on the same
    model.  Excluded ("unsure") pixels: equal keys within `tie` (oracle key_margin) or an
    owner -- on either side -- whose fp64 gate quantity lies within `tie` of a threshold
    (oracle gate_margin).  Everything else is compared exactly: the owner map both ways,
    why bits, weights and stamps; positions within 0.05 mm, normals 1e-4, colours 1e-5;
    lifted points pixel by pixel (the row-major lift order of both sides)."""
    n = ids.shape[0]
    gown = np.where(owner >= 0, ids[np.maximum(owner, 0)], -1)
    oown = o["owner"]
    unsure_pt = o["gate_margin"] <= tie

    def unsure_owner(own):
        return (own >= 0) & unsure_pt[np.maximum(own, 0)]

    excl = (o["key_margin"] <= tie) | unsure_owner(gown) | unsure_owner(oown)
    assert excl.mean() < 1e-3, excl.mean()
    bad = np.flatnonzero((gown != oown) & ~excl)
    assert bad.size == 0, (bad[:10], gown[bad[:10]], oown[bad[:10]])
    sure = ~unsure_pt[ids]
    wbad = np.flatnonzero(sure & (why != o["why"][ids]))
    assert wbad.size == 0, (wbad[:10], why[wbad[:10]], o["why"][ids][wbad[:10]])
    assert stats[0] == int((gown >= 0).sum())
    # the model after the fusion, matched by caller id
    mod = M.mis_get_model(ctx.ptr, k)
    gid = mod["ids"]
    aff = np.unique(np.concatenate([gown[excl], oown[excl]]))
    old = gid < n
    ok = old & ~np.isin(gid, aff)
    go = gid[ok]
    assert (mod["weight"][ok] == o["weight"][go]).all()
    assert (mod["stamp"][ok] == o["stamp"][go]).all()
    assert np.abs(mod["xyz"][ok] - o["xyz"][go]).max() < 0.05
    assert np.abs(mod["nrm"][ok] - o["nrm"][go]).max() < 1e-4
    assert np.abs(mod["rgb"][ok] - o["rgb"][go]).max() < 1e-5
    fused = ok & (mod["stamp"] == frame_index) & np.isin(gid, gown[gown >= 0])
    assert fused.sum() > 0
    # lifted points: GPU id n + r <-> the r-th lifted pixel of the GPU owner map (row-major)
    _, _, dv, nv = O.frame_prep(fr)
    valid = (dv & nv).ravel().astype(bool)
    g_lift = np.flatnonzero(valid & (gown < 0))
    o_lift = np.flatnonzero(valid & (oown < 0))
    assert np.isin(np.setxor1d(g_lift, o_lift), np.flatnonzero(excl)).all()
    assert n_out == n + g_lift.size and stats[1] == g_lift.size
    new = ~old
    r_g = gid[new] - n
    pix_g = g_lift[r_g]
    both = np.isin(pix_g, o_lift)
    r_o = np.searchsorted(o_lift, pix_g[both])
    sel = np.flatnonzero(new)[both]
    assert np.abs(mod["xyz"][sel] - o["xyz"][n + r_o]).max() < 1e-3
    assert np.abs(mod["nrm"][sel] - o["nrm"][n + r_o]).max() < 1e-5
    assert (mod["rgb"][sel] == o["rgb"][n + r_o]).all()
    assert (mod["weight"][new] == 1).all() and (mod["stamp"][new] == frame_index).all()
    lm = o["lift_margin"][r_o] > 1e-5
    oi = np.sort(o["lift_idx"][r_o], axis=1)
    assert (mod["knn_idx"][sel][lm] == oi[lm]).all()
    return mod
