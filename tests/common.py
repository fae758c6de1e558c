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
