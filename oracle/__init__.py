"""ctypes front-end of the fp64 CPU oracle (oracle.cpp).

TEST INFRASTRUCTURE ONLY: import this from tests/, __graft_entry__.smoke() or
bench.py's cpu_baseline / ``--impl reference`` legs, never from the product
package.  It shares no code with the CUDA path.

Every function takes plain numpy arrays (float32 inputs exactly as the CUDA
path receives them) and returns float64 results.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (fp64, no -ffast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-fopenmp",
                               _SRC, "-o", _SO + ".tmp"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


class or_params(C.Structure):
    _fields_ = [("k", C.c_int32), ("n_nbr", C.c_int32),
                ("w_data", C.c_double), ("w_pt", C.c_double), ("w_reg", C.c_double), ("w_corr", C.c_double),
                ("eps_d", C.c_double), ("eps_n_deg", C.c_double),
                ("tau_z", C.c_double), ("delta_deg", C.c_double), ("trunc", C.c_double), ("omega_max", C.c_double),
                ("gn_iters", C.c_int32), ("pcg_iters", C.c_int32), ("lambda_", C.c_double),
                ("solve_mode", C.c_int32), ("lm", C.c_int32), ("lm_mu0", C.c_double),
                ("joint_pose", C.c_int32), ("w_r", C.c_double), ("w_p", C.c_double), ("w_rot", C.c_double)]


class or_frame(C.Structure):
    _fields_ = [("W", C.c_int32), ("H", C.c_int32),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("depth", C.c_void_p), ("pose", C.c_double * 12)]


class or_problem(C.Structure):
    _fields_ = [("n", C.c_int64), ("xyz", C.c_void_p), ("nrm", C.c_void_p),
                ("idx", C.c_void_p), ("w", C.c_void_p),
                ("m", C.c_int32), ("g", C.c_void_p), ("nbr", C.c_void_p),
                ("nf", C.c_int32), ("fsrc", C.c_void_p), ("fdst", C.c_void_p)]


class or_model(C.Structure):
    _fields_ = [("n", C.c_int64), ("xyz", C.c_void_p), ("nrm", C.c_void_p), ("rgb", C.c_void_p),
                ("weight", C.c_void_p), ("stamp", C.c_void_p)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            P = C.POINTER
            L.or_frame_prep.argtypes = [P(or_frame), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_skin.argtypes = [C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                  C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_exp.argtypes = [C.c_void_p, C.c_void_p]
            L.or_set_threads.argtypes = [C.c_int32]
            L.or_warp.argtypes = [P(or_problem), C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_associate.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_system.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_int64,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_system.restype = C.c_int64
            L.or_residuals.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
            L.or_residuals.restype = C.c_int64
            L.or_solve.argtypes = [C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_double, C.c_int32, C.c_int32, C.c_void_p]
            L.or_solve.restype = C.c_int32
            L.or_register.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_system_pose.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_int64,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_system_pose.restype = C.c_int64
            L.or_residuals_pose.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
            L.or_residuals_pose.restype = C.c_int64
            L.or_register_pose.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_euler_zyx.argtypes = [C.c_void_p, C.c_void_p]
            L.or_pose_prior.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_pose_prior.restype = C.c_int32
            L.or_warp_aff.argtypes = [P(or_problem), C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_associate_aff.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_rot.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_system_aff.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
            L.or_system_aff.restype = C.c_int64
            L.or_residuals_aff.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
            L.or_residuals_aff.restype = C.c_int64
            L.or_solve_aff.argtypes = [C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_double, C.c_int32, C.c_int32, C.c_void_p]
            L.or_solve_aff.restype = C.c_int32
            L.or_register_aff.argtypes = [P(or_params), P(or_problem), P(or_frame), C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
            L.or_warp_model_aff.argtypes = [P(or_problem), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_warp_model.argtypes = [P(or_problem), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.or_fuse.argtypes = [P(or_params), P(or_model), P(or_frame), C.c_void_p, C.c_int32, C.c_int32,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p]
            L.or_fuse.restype = C.c_int64
            L.or_filter.argtypes = [C.c_int64] + [C.c_void_p] * 6 + [C.c_float, C.c_int32, C.c_int32, C.c_float,
                                                                      C.c_float] + [C.c_void_p] * 8
            L.or_filter.restype = C.c_int64
            L.or_regenerate_nodes.argtypes = [C.c_int64, C.c_void_p, C.c_float, C.c_int32, C.c_void_p, C.c_void_p,
                                              C.c_void_p]
            L.or_regenerate_nodes.restype = C.c_int64
            _lib = L
    return _lib


# ---------------------------------------------------------------- marshalling
def _p(a):
    return None if a is None else a.ctypes.data


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


PAPER_DEFAULTS = dict(k=4, n_nbr=4, w_data=1.0, w_pt=1.0, w_reg=1e4, w_corr=10.0,
                      eps_d=15.0, eps_n_deg=10.0, tau_z=10.0, delta_deg=10.0, trunc=40.0, omega_max=10.0,
                      gn_iters=5, pcg_iters=10, lambda_=1e-4, solve_mode=1, lm=0, lm_mu0=1e-3,
                      joint_pose=0, w_r=1e6, w_p=1000.0, w_rot=1000.0)


def set_threads(n: int) -> None:
    """Host threads of the oracle (bench.py's all-cores column; default 1)."""
    lib().or_set_threads(int(n))


def params(**kw) -> or_params:
    d = dict(PAPER_DEFAULTS)
    d.update(kw)
    return or_params(**d)


class Frame:
    """Owns the arrays an or_frame points to."""

    def __init__(self, depth, intr, pose):
        self.depth = _f32(depth)
        H, W = self.depth.shape
        self.s = or_frame(W, H, intr["fx"], intr["fy"], intr["cx"], intr["cy"], _p(self.depth),
                          (C.c_double * 12)(*[float(x) for x in np.asarray(pose, np.float64).ravel()]))


class Problem:
    def __init__(self, xyz, nrm, idx, w, g, nbr, fsrc=None, fdst=None):
        self.xyz, self.nrm = _f32(xyz), _f32(nrm)
        self.idx, self.w = _i32(idx), _f32(w)
        self.g, self.nbr = _f32(g), _i32(nbr)
        self.k = self.idx.shape[1]
        self.n_nbr = self.nbr.shape[1]
        self.fsrc = _f32(fsrc if fsrc is not None else np.zeros((0, 3)))
        self.fdst = _f32(fdst if fdst is not None else np.zeros((0, 3)))
        self.s = or_problem(self.xyz.shape[0], _p(self.xyz), _p(self.nrm), _p(self.idx), _p(self.w),
                            self.g.shape[0], _p(self.g), _p(self.nbr),
                            self.fsrc.shape[0], _p(self.fsrc), _p(self.fdst))


def identity_state(m):
    Rt = np.zeros((m, 12))
    Rt[:, 0] = Rt[:, 4] = Rt[:, 8] = 1.0
    return Rt


def frame_prep(fr: Frame):
    H, W = fr.depth.shape
    q = np.zeros((H, W, 3)); N = np.zeros((H, W, 3))
    dv = np.zeros((H, W), np.uint8); nv = np.zeros((H, W), np.uint8)
    lib().or_frame_prep(C.byref(fr.s), _p(q), _p(N), _p(dv), _p(nv))
    return q, N, dv.astype(bool), nv.astype(bool)


def skin(points, g, k):
    points, g = _f32(points), _f32(g)
    n = points.shape[0]
    idx = np.zeros((n, k), np.int32); w = np.zeros((n, k)); mg = np.zeros(n)
    lib().or_skin(n, _p(points), g.shape[0], _p(g), k, _p(idx), _p(w), _p(mg))
    return idx, w, mg


def exp_so3(w):
    w = np.ascontiguousarray(w, np.float64); R = np.zeros(9)
    lib().or_exp(_p(w), _p(R))
    return R.reshape(3, 3)


def warp(pb: Problem, Rt, pose):
    n = pb.xyz.shape[0]
    Rt = np.ascontiguousarray(Rt, np.float64); pose = np.ascontiguousarray(pose, np.float64)
    xh = np.zeros((n, 3)); nh = np.zeros((n, 3)); vt = np.zeros((n, 3)); nt = np.zeros((n, 3))
    ok = np.zeros(n, np.uint8)
    lib().or_warp(C.byref(pb.s), pb.k, _p(Rt), _p(pose), _p(xh), _p(nh), _p(vt), _p(nt), _p(ok))
    return xh, nh, vt, nt, ok.astype(bool)


def associate(prm: or_params, pb: Problem, fr: Frame, Rt):
    n = pb.xyz.shape[0]
    Rt = np.ascontiguousarray(Rt, np.float64)
    pix = np.zeros(n, np.int32); why = np.zeros(n, np.uint8); mg = np.zeros(n)
    lib().or_associate(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(pix), _p(why), _p(mg))
    return pix, why, mg


def feature_skin(pb: Problem):
    if pb.fsrc.shape[0] == 0:
        return np.zeros((0, pb.k), np.int32), np.zeros((0, pb.k)), np.zeros(0)
    return skin(pb.fsrc, pb.g, pb.k)


def system(prm: or_params, pb: Problem, fr: Frame, Rt, fskin=None):
    """Returns dict(blocks={(j,l): 6x6}, rows, cols, vals, rhs, energy, n_assoc)."""
    m = pb.g.shape[0]
    Rt = np.ascontiguousarray(Rt, np.float64)
    fidx, fw = (fskin if fskin is not None else feature_skin(pb)[:2])
    fidx = _i32(fidx.reshape(-1, pb.k)); fw = np.ascontiguousarray(fw, np.float64)
    rhs = np.zeros(6 * m); E = np.zeros(5); na = np.zeros(1, np.int64)
    cap = 0
    z = np.zeros(1, np.int32); zd = np.zeros(36)
    nb = lib().or_system(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(fidx), _p(fw), cap,
                         _p(z), _p(z), _p(zd), _p(rhs), _p(E), _p(na))
    rows = np.zeros(nb, np.int32); cols = np.zeros(nb, np.int32); vals = np.zeros((nb, 36))
    lib().or_system(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(fidx), _p(fw), nb,
                    _p(rows), _p(cols), _p(vals), _p(rhs), _p(E), _p(na))
    return dict(rows=rows, cols=cols, vals=vals.reshape(nb, 6, 6), rhs=rhs, energy=E, n_assoc=int(na[0]))


def dense_H(sysd, m):
    H = np.zeros((6 * m, 6 * m))
    for r, c, B in zip(sysd["rows"], sysd["cols"], sysd["vals"]):
        H[6 * r:6 * r + 6, 6 * c:6 * c + 6] += B
        if r != c:
            H[6 * c:6 * c + 6, 6 * r:6 * r + 6] += B.T
    return H


def residuals(prm: or_params, pb: Problem, fr: Frame, Rt, pix_frozen, fskin=None):
    m = pb.g.shape[0]
    Rt = np.ascontiguousarray(Rt, np.float64)
    fidx, fw = (fskin if fskin is not None else feature_skin(pb)[:2])
    fidx = _i32(fidx.reshape(-1, pb.k)); fw = np.ascontiguousarray(fw, np.float64)
    pix_frozen = _i32(pix_frozen)
    cap = 4 * pb.xyz.shape[0] + 3 * m * pb.n_nbr + 3 * pb.fsrc.shape[0]
    r = np.zeros(cap); J = np.zeros((cap, 6 * m))
    nr = lib().or_residuals(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(pix_frozen), _p(fidx), _p(fw),
                            cap, _p(r), _p(J))
    assert nr >= 0
    return r[:nr], J[:nr]


def solve(sysd, m, lam, mode, pcg_iters):
    x = np.zeros(6 * m)
    nb = len(sysd["rows"])
    vals = np.ascontiguousarray(sysd["vals"].reshape(nb, 36), np.float64)
    it = lib().or_solve(m, nb, _p(_i32(sysd["rows"])), _p(_i32(sysd["cols"])), _p(vals),
                        _p(np.ascontiguousarray(sysd["rhs"], np.float64)), lam, mode, pcg_iters, _p(x))
    return x, it


def register(prm: or_params, pb: Problem, fr: Frame, Rt0=None, with_accepted=False):
    m = pb.g.shape[0]
    Rt = identity_state(m) if Rt0 is None else np.array(Rt0, np.float64, copy=True)
    G = prm.gn_iters
    E = np.zeros((G + 1, 5)); na = np.zeros(G + 1, np.int64)
    acc = np.zeros(G + 1, np.int32)
    lib().or_register(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(E), _p(na), _p(acc))
    if with_accepted:
        return Rt, E, na, acc
    return Rt, E, na


# ---------------------------------------------------------------- NEXT-2: joint global pose
def euler_zyx(O):
    """ZYX Euler angles (yaw, pitch, roll) of a rotation matrix O = Rz Ry Rx."""
    e = np.zeros(3)
    lib().or_euler_zyx(_p(np.ascontiguousarray(O, np.float64).reshape(9)), _p(e))
    return e


def pose_prior(prior, cur):
    """Eq. 10 residuals r (6) and Jacobian J (6x6) w.r.t. [dphi, dtau] (A37-A39); flag 1 = gimbal lock."""
    r = np.zeros(6); J = np.zeros(36)
    fl = lib().or_pose_prior(_p(np.ascontiguousarray(prior, np.float64)), _p(np.ascontiguousarray(cur, np.float64)),
                             _p(r), _p(J))
    return r, J.reshape(6, 6), int(fl)


def system_pose(prm: or_params, pb: Problem, fr: Frame, Rt, pose_cur, fskin=None):
    """Joint system over m + 1 unknowns (the pose last); energy[7]."""
    m = pb.g.shape[0]
    Rt = np.ascontiguousarray(Rt, np.float64)
    pc = np.ascontiguousarray(pose_cur, np.float64)
    fidx, fw = (fskin if fskin is not None else feature_skin(pb)[:2])
    fidx = _i32(fidx.reshape(-1, pb.k)); fw = np.ascontiguousarray(fw, np.float64)
    rhs = np.zeros(6 * (m + 1)); E = np.zeros(7); na = np.zeros(1, np.int64)
    z = np.zeros(1, np.int32); zd = np.zeros(36)
    nb = lib().or_system_pose(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(pc), _p(fidx), _p(fw), 0,
                              _p(z), _p(z), _p(zd), _p(rhs), _p(E), _p(na))
    rows = np.zeros(nb, np.int32); cols = np.zeros(nb, np.int32); vals = np.zeros((nb, 36))
    lib().or_system_pose(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(pc), _p(fidx), _p(fw), nb,
                         _p(rows), _p(cols), _p(vals), _p(rhs), _p(E), _p(na))
    return dict(rows=rows, cols=cols, vals=vals.reshape(nb, 6, 6), rhs=rhs, energy=E, n_assoc=int(na[0]))


def residuals_pose(prm: or_params, pb: Problem, fr: Frame, Rt, pose_cur, pix_frozen, fskin=None):
    m = pb.g.shape[0]
    Rt = np.ascontiguousarray(Rt, np.float64)
    pc = np.ascontiguousarray(pose_cur, np.float64)
    fidx, fw = (fskin if fskin is not None else feature_skin(pb)[:2])
    fidx = _i32(fidx.reshape(-1, pb.k)); fw = np.ascontiguousarray(fw, np.float64)
    pix_frozen = _i32(pix_frozen)
    cap = 4 * pb.xyz.shape[0] + 3 * m * pb.n_nbr + 3 * pb.fsrc.shape[0] + 6
    r = np.zeros(cap); J = np.zeros((cap, 6 * (m + 1)))
    nr = lib().or_residuals_pose(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(pc), _p(pix_frozen),
                                 _p(fidx), _p(fw), cap, _p(r), _p(J))
    assert nr >= 0
    return r[:nr], J[:nr]


def register_pose(prm: or_params, pb: Problem, fr: Frame, Rt0=None, pose0=None, with_accepted=False):
    """Joint registration: returns (Rt, pose, E (G+1 x 7), n_assoc[, accepted]); pose0 defaults to the prior."""
    m = pb.g.shape[0]
    Rt = identity_state(m) if Rt0 is None else np.array(Rt0, np.float64, copy=True)
    pose = np.array(fr.s.pose[:] if pose0 is None else pose0, np.float64)
    G = prm.gn_iters
    E = np.zeros((G + 1, 7)); na = np.zeros(G + 1, np.int64)
    acc = np.zeros(G + 1, np.int32)
    lib().or_register_pose(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(Rt), _p(pose), _p(E), _p(na), _p(acc))
    if with_accepted:
        return Rt, pose, E, na, acc
    return Rt, pose, E, na


# ---------------------------------------------------------------- NEXT-4: affine nodes + E_rot
def identity_affine(m):
    """m x 12 affine state: A_j = I (row-major), t_j = 0."""
    return identity_state(m)


def rot_terms(A):
    """Eq. 5 residuals (6) and their Jacobian (6 x 9, A row-major)."""
    r = np.zeros(6); J = np.zeros(54)
    lib().or_rot(_p(np.ascontiguousarray(A, np.float64).reshape(9)), _p(r), _p(J))
    return r, J.reshape(6, 9)


def warp_aff(pb: Problem, At, pose):
    n = pb.xyz.shape[0]
    At = np.ascontiguousarray(At, np.float64)
    out = [np.zeros((n, 3)) for _ in range(4)]
    ok = np.zeros(n, np.uint8)
    lib().or_warp_aff(C.byref(pb.s), pb.k, _p(At), _p(np.ascontiguousarray(pose, np.float64)),
                      *[_p(o) for o in out], _p(ok))
    return (*out, ok)


def associate_aff(prm: or_params, pb: Problem, fr: Frame, At):
    n = pb.xyz.shape[0]
    At = np.ascontiguousarray(At, np.float64)
    pix = np.zeros(n, np.int32); why = np.zeros(n, np.uint8); mg = np.zeros(n)
    lib().or_associate_aff(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(At), _p(pix), _p(why), _p(mg))
    return pix, why, mg


def system_aff(prm: or_params, pb: Problem, fr: Frame, At, fskin=None):
    """12 x 12 block normal equations of the affine model; energy[6]."""
    m = pb.g.shape[0]
    At = np.ascontiguousarray(At, np.float64)
    fidx, fw = (fskin if fskin is not None else feature_skin(pb)[:2])
    fidx = _i32(fidx.reshape(-1, pb.k)); fw = np.ascontiguousarray(fw, np.float64)
    rhs = np.zeros(12 * m); E = np.zeros(6); na = np.zeros(1, np.int64)
    z = np.zeros(1, np.int32); zd = np.zeros(144)
    nb = lib().or_system_aff(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(At), _p(fidx), _p(fw), 0,
                             _p(z), _p(z), _p(zd), _p(rhs), _p(E), _p(na))
    rows = np.zeros(nb, np.int32); cols = np.zeros(nb, np.int32); vals = np.zeros((nb, 144))
    lib().or_system_aff(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(At), _p(fidx), _p(fw), nb,
                        _p(rows), _p(cols), _p(vals), _p(rhs), _p(E), _p(na))
    return dict(rows=rows, cols=cols, vals=vals.reshape(nb, 12, 12), rhs=rhs, energy=E, n_assoc=int(na[0]))


def dense_H_aff(sysd, m):
    H = np.zeros((12 * m, 12 * m))
    for r, c, B in zip(sysd["rows"], sysd["cols"], sysd["vals"]):
        H[12 * r:12 * r + 12, 12 * c:12 * c + 12] += B
        if r != c:
            H[12 * c:12 * c + 12, 12 * r:12 * r + 12] += B.T
    return H


def residuals_aff(prm: or_params, pb: Problem, fr: Frame, At, pix_frozen, fskin=None):
    m = pb.g.shape[0]
    At = np.ascontiguousarray(At, np.float64)
    fidx, fw = (fskin if fskin is not None else feature_skin(pb)[:2])
    fidx = _i32(fidx.reshape(-1, pb.k)); fw = np.ascontiguousarray(fw, np.float64)
    cap = 4 * pb.xyz.shape[0] + 3 * m * pb.n_nbr + 3 * pb.fsrc.shape[0] + 6 * m
    r = np.zeros(cap); J = np.zeros((cap, 12 * m))
    nr = lib().or_residuals_aff(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(At), _p(_i32(pix_frozen)), _p(fidx),
                                _p(fw), cap, _p(r), _p(J))
    assert nr >= 0
    return r[:nr], J[:nr]


def solve_aff(sysd, m, lam, mode, pcg_iters):
    x = np.zeros(12 * m)
    nb = len(sysd["rows"])
    vals = np.ascontiguousarray(sysd["vals"].reshape(nb, 144), np.float64)
    it = lib().or_solve_aff(m, nb, _p(_i32(sysd["rows"])), _p(_i32(sysd["cols"])), _p(vals),
                            _p(np.ascontiguousarray(sysd["rhs"], np.float64)), lam, mode, pcg_iters, _p(x))
    return x, it


def register_aff(prm: or_params, pb: Problem, fr: Frame, At0=None, with_accepted=False):
    """Affine-node Gauss-Newton (or LM with prm.lm): returns (At, E (G+1 x 6), n_assoc[, accepted])."""
    m = pb.g.shape[0]
    At = identity_affine(m) if At0 is None else np.array(At0, np.float64, copy=True)
    G = prm.gn_iters
    E = np.zeros((G + 1, 6)); na = np.zeros(G + 1, np.int64); acc = np.zeros(G + 1, np.int32)
    lib().or_register_aff(C.byref(prm), C.byref(pb.s), C.byref(fr.s), _p(At), _p(E), _p(na), _p(acc))
    if with_accepted:
        return At, E, na, acc
    return At, E, na


def warp_model_aff(pb: Problem, At):
    n, m = pb.xyz.shape[0], pb.g.shape[0]
    At = np.ascontiguousarray(At, np.float64)
    xyz = np.zeros((n, 3)); nrm = np.zeros((n, 3)); g = np.zeros((m, 3))
    lib().or_warp_model_aff(C.byref(pb.s), pb.k, _p(At), _p(xyz), _p(nrm), _p(g))
    return xyz, nrm, g


def warp_model(pb: Problem, Rt):
    n, m = pb.xyz.shape[0], pb.g.shape[0]
    Rt = np.ascontiguousarray(Rt, np.float64)
    xyz = np.zeros((n, 3)); nrm = np.zeros((n, 3)); g = np.zeros((m, 3))
    lib().or_warp_model(C.byref(pb.s), pb.k, _p(Rt), _p(xyz), _p(nrm), _p(g))
    return xyz, nrm, g


def fuse(prm: or_params, xyz, nrm, rgb, weight, stamp, fr: Frame, rgb_obs, frame_index, g):
    xyz, nrm, rgb, weight = _f32(xyz), _f32(nrm), _f32(rgb), _f32(weight)
    stamp = _i32(stamp); g = _f32(g)
    n = xyz.shape[0]
    H, W = fr.depth.shape
    cap = n + H * W
    k = prm.k
    md = or_model(n, _p(xyz), _p(nrm), _p(rgb), _p(weight), _p(stamp))
    ro = None if rgb_obs is None else _f32(rgb_obs)
    out = dict(xyz=np.zeros((cap, 3)), nrm=np.zeros((cap, 3)), rgb=np.zeros((cap, 3)),
               weight=np.zeros(cap), stamp=np.zeros(cap, np.int32),
               lift_idx=np.zeros((H * W, k), np.int32), lift_w=np.zeros((H * W, k)), lift_margin=np.zeros(H * W),
               owner=np.zeros(H * W, np.int64), key_margin=np.zeros(H * W), why=np.zeros(n, np.uint8),
               gate_margin=np.zeros(n))
    nl = lib().or_fuse(C.byref(prm), C.byref(md), C.byref(fr.s), _p(ro), frame_index, g.shape[0], _p(g),
                       _p(out["xyz"]), _p(out["nrm"]), _p(out["rgb"]), _p(out["weight"]), _p(out["stamp"]),
                       _p(out["lift_idx"]), _p(out["lift_w"]), _p(out["lift_margin"]),
                       _p(out["owner"]), _p(out["key_margin"]), _p(out["why"]), _p(out["gate_margin"]))
    for key in ("xyz", "nrm", "rgb", "weight", "stamp"):
        out[key] = out[key][:n + nl]
    for key in ("lift_idx", "lift_w", "lift_margin"):
        out[key] = out[key][:nl]
    out["n_lift"] = int(nl)
    return out


def filter_points(xyz, nrm, rgb, weight, stamp, ids, grid, frame_index, tau_time, tau_weight, omega_max):
    """O7: Alg. 3 downsampling + deletion (readings A30-A34)."""
    xyz, nrm, rgb, weight = _f32(xyz), _f32(nrm), _f32(rgb), _f32(weight)
    stamp = _i32(stamp)
    ids = None if ids is None else np.ascontiguousarray(ids, np.int64)
    n = xyz.shape[0]
    out = dict(xyz=np.zeros((n, 3)), nrm=np.zeros((n, 3)), rgb=np.zeros((n, 3)), weight=np.zeros(n),
               stamp=np.zeros(n, np.int32), ids=np.zeros(n, np.int64), stable=np.zeros(n, np.uint8))
    cells = C.c_int64(0)
    no = lib().or_filter(n, _p(xyz), _p(nrm), _p(rgb), _p(weight), _p(stamp), _p(ids), float(grid), int(frame_index),
                         int(tau_time), float(tau_weight), float(omega_max), _p(out["xyz"]), _p(out["nrm"]),
                         _p(out["rgb"]), _p(out["weight"]), _p(out["stamp"]), _p(out["ids"]), _p(out["stable"]),
                         C.addressof(cells))
    for key in list(out):
        out[key] = out[key][:no]
    out["cells"] = int(cells.value)
    return out


def regenerate_nodes(xyz, grid, n_nbr):
    """O8: Alg. 2 Step 5 node regeneration (reading A36).
    Returns (g (m x 3, fp64 centroids), nbr (m x n_nbr), nbr_margin (m))."""
    xyz = _f32(xyz)
    n = xyz.shape[0]
    g = np.zeros((max(n, 1), 3))
    nbr = np.zeros((max(n, 1), max(n_nbr, 1)), np.int32)
    mg = np.zeros(max(n, 1))
    m = lib().or_regenerate_nodes(n, _p(xyz), float(grid), int(n_nbr), _p(g), _p(nbr), _p(mg))
    return g[:m], nbr[:m, :n_nbr], mg[:m]
