"""Thin ctypes binding of libmis.so (include/mis.h) -- argument marshalling only.

Every step of the registration / fusion path runs in the CUDA kernels of
libmis.so; this module only converts numpy arrays (host, MIS_MEM_HOST) or torch
CUDA tensors (device, MIS_MEM_DEVICE) into pointers, calls the C entry point of
the same name and raises MisError on a non-zero status.  There is no CPU
fallback: importing fails loudly when libmis.so is missing.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MIS_LIB_PATH", os.path.join(_HERE, "libmis.so"))   # override: experiments only

MIS_MEM_HOST, MIS_MEM_DEVICE = 0, 1
MIS_MAX_GN, MIS_MAX_K = 32, 8
MIS_F_FINAL_ENERGY, MIS_F_GRID_SOLVER, MIS_F_STANDARD_PCG = 1, 4, 8
MIS_F_LM = 16   # Levenberg-Marquardt (include/mis.h)
MIS_F_JOINT_POSE = 32   # NEXT-2 joint global pose (include/mis.h)
MIS_F_AFFINE = 64   # NEXT-4 affine nodes + E_rot (include/mis.h)
STATUS = {0: "MIS_OK", 1: "MIS_E_ARG", 2: "MIS_E_STATE", 3: "MIS_E_CUDA", 4: "MIS_E_NCCL",
          5: "MIS_E_NOMEM", 6: "MIS_E_CAPACITY", 7: "MIS_E_NUMERIC"}


class MisError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class mis_params(C.Structure):
    _fields_ = [("k", C.c_int32), ("n_nbr", C.c_int32),
                ("w_data", C.c_float), ("w_point", C.c_float), ("w_reg", C.c_float), ("w_corr", C.c_float),
                ("eps_d_mm", C.c_float), ("eps_n_deg", C.c_float),
                ("tau_z_mm", C.c_float), ("delta_deg", C.c_float), ("trunc_mm", C.c_float), ("omega_max", C.c_float),
                ("gn_iters", C.c_int32), ("pcg_iters", C.c_int32), ("lambda_", C.c_float), ("flags", C.c_uint32),
                ("w_r", C.c_float), ("w_p", C.c_float), ("w_rot", C.c_float)]


class mis_intrinsics(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class mis_report(C.Structure):
    _fields_ = [("iters", C.c_int32), ("status", C.c_int32),
                ("energy", (C.c_double * 5) * (MIS_MAX_GN + 1)),
                ("n_assoc", C.c_int64 * (MIS_MAX_GN + 1)),
                ("pcg_rel_res", C.c_float * MIS_MAX_GN),
                ("nnzb", C.c_int64), ("n_segments", C.c_int64), ("solver_cluster", C.c_int32),
                ("reserved", C.c_int32), ("n_guard", C.c_int64 * (MIS_MAX_GN + 1)),
                ("energy_pose", (C.c_double * 2) * (MIS_MAX_GN + 1)),
                ("energy_rot", C.c_double * (MIS_MAX_GN + 1))]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1803_02009_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)
_P, _V = C.POINTER, C.c_void_p
_sig = {
    "mis_abi_version": ([], C.c_int32),
    "mis_default_params": ([_P(mis_params)], None),
    "mis_create": ([_P(mis_params), C.c_int, _V, C.c_int, C.c_int, _V, _P(_V)], C.c_int),
    "mis_destroy": ([_V], C.c_int),
    "mis_last_error": ([_V], C.c_char_p),
    "mis_nccl_unique_id": ([_V], C.c_int),
    "mis_set_params": ([_V, _P(mis_params)], C.c_int),
    "mis_workspace_bytes": ([_V, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _P(C.c_size_t)], C.c_int),
    "mis_bind_workspace": ([_V, _V, C.c_size_t], C.c_int),
    "mis_set_model": ([_V, C.c_int64, C.c_int, _V, _V, _V, _V, _V, _V, C.c_int64], C.c_int),
    "mis_set_graph": ([_V, C.c_int32, C.c_int, _V, _V, _V, _V], C.c_int),
    "mis_set_frame": ([_V, C.c_int, _V, _P(mis_intrinsics), _V], C.c_int),
    "mis_set_features": ([_V, C.c_int, C.c_int32, _V, _V], C.c_int),
    "mis_register": ([_V, C.c_int, _V, _P(mis_intrinsics), _V, C.c_int32, _V, _V, _P(mis_report)], C.c_int),
    "mis_get_nodes": ([_V, C.c_int, _V], C.c_int),
    "mis_get_nodes_f64": ([_V, _V], C.c_int),
    "mis_get_graph": ([_V, C.c_int, _V], C.c_int),
    "mis_get_pose": ([_V, _V], C.c_int),
    "mis_dbg_set_pose": ([_V, _V], C.c_int),
    "mis_get_nbr": ([_V, C.c_int, _V], C.c_int),
    "mis_warp": ([_V, C.c_int, _V, _V], C.c_int),
    "mis_fuse": ([_V, C.c_int, _V, C.c_int32, _P(C.c_int64), _V], C.c_int),
    "mis_stage_colour": ([_V, _V], C.c_int),
    "mis_filter": ([_V, C.c_float, C.c_int32, C.c_int32, C.c_float, _P(C.c_int64), _V], C.c_int),
    "mis_regenerate_nodes": ([_V, C.c_float, _P(C.c_int32)], C.c_int),
    "mis_get_model": ([_V, C.c_int, _V, _V, _V, _V, _V, _V, _V, _V, _P(C.c_int64)], C.c_int),
    "mis_skin": ([_V, C.c_int, C.c_int64, _V, _V, _V], C.c_int),
    "mis_dbg_set_nodes": ([_V, C.c_int, _V], C.c_int),
    "mis_dbg_frame": ([_V, C.c_int, _V], C.c_int),
    "mis_dbg_associate": ([_V, C.c_int, _V, _V], C.c_int),
    "mis_dbg_system": ([_V, _V, _V, _V, _V, _V, _P(C.c_int64)], C.c_int),
    "mis_dbg_fuse_register": ([_V, _V, _V], C.c_int),
    "mis_prof_name": ([C.c_int], C.c_char_p),
    "mis_prof_enable": ([_V, C.c_int], C.c_int),
    "mis_prof_read": ([_V, _V, _V, C.c_int], C.c_int),
    "mis_launch_count": ([], C.c_int64),
    "mis_dbg_solver_phases": ([_V, _V], C.c_int),
}
MIS_PROF_NCAT = 16
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res
EXPORTED = tuple(_sig)


# ------------------------------------------------------------------ marshalling
def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _mem_of(*arrays):
    kinds = {MIS_MEM_DEVICE if (_is_torch(a) and a.is_cuda) else MIS_MEM_HOST for a in arrays if a is not None}
    if len(kinds) > 1:
        raise ValueError("all array arguments of one call must be host (numpy / CPU tensor) or device alike")
    return kinds.pop() if kinds else MIS_MEM_HOST


def _ptr(x, dtype=None):
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise ValueError("tensor arguments must be contiguous")
        return C.c_void_p(x.data_ptr())
    if dtype is not None and x.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {x.dtype}")
    if not x.flags["C_CONTIGUOUS"]:
        raise ValueError("host arguments must be C-contiguous")
    return C.c_void_p(x.ctypes.data)


def _check(ctx, st):
    if st != 0:
        msg = _lib.mis_last_error(ctx).decode() if ctx else ""
        raise MisError(st, msg)


def mis_default_params(**overrides) -> mis_params:
    p = mis_params()
    _lib.mis_default_params(C.byref(p))
    for k, v in overrides.items():
        setattr(p, "lambda_" if k == "lambda" else k, v)
    return p


def intrinsics(fx, fy, cx, cy, width, height) -> mis_intrinsics:
    return mis_intrinsics(fx, fy, cx, cy, width, height)


def mis_abi_version():
    return _lib.mis_abi_version()


def mis_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(None, _lib.mis_nccl_unique_id(buf))
    return buf.raw


def mis_create(params: mis_params, device=0, stream=None, rank=0, world=1, nccl_id: bytes | None = None):
    ctx = C.c_void_p()
    sid = None if stream is None else C.c_void_p(stream)
    nid = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
    st = _lib.mis_create(C.byref(params), device, sid, rank, world, nid, C.byref(ctx))
    if st != 0:
        raise MisError(st, "mis_create failed (is a CUDA device present?)")
    return ctx


def mis_destroy(ctx):
    _check(ctx, _lib.mis_destroy(ctx))


def mis_set_params(ctx, params):
    _check(ctx, _lib.mis_set_params(ctx, C.byref(params)))


def mis_workspace_bytes(ctx, n_cap, m, H, W) -> int:
    b = C.c_size_t()
    _check(ctx, _lib.mis_workspace_bytes(ctx, int(n_cap), int(m), int(H), int(W), C.byref(b)))
    return int(b.value)


def mis_bind_workspace(ctx, buf):
    """buf: a contiguous CUDA tensor (e.g. torch.empty(bytes, dtype=torch.uint8, device='cuda'))."""
    _check(ctx, _lib.mis_bind_workspace(ctx, _ptr(buf), int(buf.numel() * buf.element_size())))


def mis_set_model(ctx, xyz, nrm, rgb=None, weight=None, stamp=None, ids=None, capacity=None):
    n = int(xyz.shape[0])
    mem = _mem_of(xyz, nrm, rgb, weight, stamp, ids)
    cap = n if capacity is None else int(capacity)
    _check(ctx, _lib.mis_set_model(ctx, n, mem, _ptr(xyz, np.float32), _ptr(nrm, np.float32), _ptr(rgb, np.float32),
                                   _ptr(weight, np.float32), _ptr(stamp, np.int32), _ptr(ids, np.int64), cap))


def mis_set_graph(ctx, node_pos, node_nbr, knn_idx=None, knn_w=None):
    mem = _mem_of(node_pos, node_nbr, knn_idx, knn_w)
    _check(ctx, _lib.mis_set_graph(ctx, int(node_pos.shape[0]), mem, _ptr(node_pos, np.float32),
                                   _ptr(node_nbr, np.int32), _ptr(knn_idx, np.int32), _ptr(knn_w, np.float32)))


def _pose_arr(pose):
    return np.ascontiguousarray(np.asarray(pose, np.float32).ravel()[:12])


def mis_set_frame(ctx, depth, intr: mis_intrinsics, pose):
    p = _pose_arr(pose)
    _check(ctx, _lib.mis_set_frame(ctx, _mem_of(depth), _ptr(depth, np.float32), C.byref(intr), _ptr(p)))


def mis_set_features(ctx, src, dst):
    mem = _mem_of(src, dst)
    _check(ctx, _lib.mis_set_features(ctx, mem, int(src.shape[0]), _ptr(src, np.float32), _ptr(dst, np.float32)))


def mis_register(ctx, depth=None, intr=None, pose=None, feat_src=None, feat_dst=None, report=True):
    mem = _mem_of(depth, feat_src, feat_dst)
    p = None if pose is None else _pose_arr(pose)
    nf = -1 if feat_src is None else int(feat_src.shape[0])
    rep = mis_report() if report else None
    st = _lib.mis_register(ctx, mem, _ptr(depth, np.float32), None if intr is None else C.byref(intr),
                           None if p is None else _ptr(p), nf, _ptr(feat_src, np.float32), _ptr(feat_dst, np.float32),
                           None if rep is None else C.byref(rep))
    _check(ctx, st)
    return rep


def report_dict(rep: mis_report):
    it = rep.iters
    return dict(iters=it, status=rep.status,
                energy=np.array([[rep.energy[i][q] for q in range(5)] for i in range(it + 1)]),
                n_assoc=np.array([rep.n_assoc[i] for i in range(it + 1)]),
                pcg_rel_res=np.array([rep.pcg_rel_res[i] for i in range(it)]),
                nnzb=rep.nnzb, n_segments=rep.n_segments, solver_cluster=rep.solver_cluster,
                n_guard=np.array([rep.n_guard[i] for i in range(it + 1)]),
                accepted=np.array([rep.n_guard[i] for i in range(it + 1)]),   # MIS_F_LM decisions
                energy_pose=np.array([[rep.energy_pose[i][q] for q in range(2)] for i in range(it + 1)]),
                energy_rot=np.array([rep.energy_rot[i] for i in range(it + 1)]))


def mis_get_nodes(ctx, out):
    _check(ctx, _lib.mis_get_nodes(ctx, _mem_of(out), _ptr(out, np.float32)))
    return out


def mis_get_nodes_f64(ctx, m):
    out = np.zeros((m, 12), np.float64)
    _check(ctx, _lib.mis_get_nodes_f64(ctx, _ptr(out)))
    return out


def mis_get_pose(ctx):
    out = np.zeros(12, np.float64)
    _check(ctx, _lib.mis_get_pose(ctx, _ptr(out)))
    return out


def mis_dbg_set_pose(ctx, pose):
    _check(ctx, _lib.mis_dbg_set_pose(ctx, _ptr(np.ascontiguousarray(pose, np.float64))))


def mis_get_graph(ctx, out):
    _check(ctx, _lib.mis_get_graph(ctx, _mem_of(out), _ptr(out, np.float32)))
    return out


def mis_get_nbr(ctx, out):
    _check(ctx, _lib.mis_get_nbr(ctx, _mem_of(out), _ptr(out, np.int32)))
    return out


def mis_warp(ctx, xyz_cam=None, nrm_cam=None):
    _check(ctx, _lib.mis_warp(ctx, _mem_of(xyz_cam, nrm_cam), _ptr(xyz_cam, np.float32), _ptr(nrm_cam, np.float32)))


def mis_fuse(ctx, rgb=None, frame_index=0):
    n_out = C.c_int64()
    stats = np.zeros(4, np.int64)
    _check(ctx, _lib.mis_fuse(ctx, _mem_of(rgb), _ptr(rgb, np.float32), frame_index, C.byref(n_out), _ptr(stats)))
    return int(n_out.value), stats


def mis_stage_colour(ctx, rgb):
    """Start the upload of the next mis_fuse's host colour now (overlapping the registration); a
    following mis_fuse(ctx, rgb) with the same host array uses the staged copy.  Host arrays only."""
    if _mem_of(rgb) != MIS_MEM_HOST:
        raise ValueError("mis_stage_colour takes a host array (device colours are read in place)")
    _check(ctx, _lib.mis_stage_colour(ctx, _ptr(rgb, np.float32)))


def mis_filter(ctx, grid_mm, frame_index, tau_time=10, tau_weight=3.0):
    """NEXT-1, Alg. 3 filtering.  Returns (n, [boxes, deleted, stable, n])."""
    n_out = C.c_int64()
    stats = np.zeros(4, np.int64)
    _check(ctx, _lib.mis_filter(ctx, grid_mm, frame_index, tau_time, tau_weight, C.byref(n_out), _ptr(stats)))
    return int(n_out.value), stats


def mis_regenerate_nodes(ctx, node_grid_mm):
    """NEXT-1, Alg. 2 Step 5 (reading A36).  Returns the new node count."""
    m = C.c_int32()
    _check(ctx, _lib.mis_regenerate_nodes(ctx, float(node_grid_mm), C.byref(m)))
    return int(m.value)


def mis_get_model(ctx, k, device=False):
    """Returns the model (internal order) as numpy arrays (or torch tensors on the device)."""
    n = C.c_int64()
    _check(ctx, _lib.mis_get_model(ctx, MIS_MEM_HOST, None, None, None, None, None, None, None, None, C.byref(n)))
    n = n.value
    if device:
        import torch
        mk = lambda shape, dt: torch.empty(shape, dtype=dt, device="cuda")  # noqa: E731
        out = dict(xyz=mk((n, 3), torch.float32), nrm=mk((n, 3), torch.float32), rgb=mk((n, 3), torch.float32),
                   weight=mk((n,), torch.float32), stamp=mk((n,), torch.int32), ids=mk((n,), torch.int64),
                   knn_idx=mk((n, k), torch.int32), knn_w=mk((n, k), torch.float32))
        mem = MIS_MEM_DEVICE
    else:
        out = dict(xyz=np.zeros((n, 3), np.float32), nrm=np.zeros((n, 3), np.float32), rgb=np.zeros((n, 3), np.float32),
                   weight=np.zeros(n, np.float32), stamp=np.zeros(n, np.int32), ids=np.zeros(n, np.int64),
                   knn_idx=np.zeros((n, k), np.int32), knn_w=np.zeros((n, k), np.float32))
        mem = MIS_MEM_HOST
    nn = C.c_int64()
    _check(ctx, _lib.mis_get_model(ctx, mem, _ptr(out["xyz"]), _ptr(out["nrm"]), _ptr(out["rgb"]), _ptr(out["weight"]),
                                   _ptr(out["stamp"]), _ptr(out["ids"]), _ptr(out["knn_idx"]), _ptr(out["knn_w"]),
                                   C.byref(nn)))
    return out


def mis_skin(ctx, pts, k):
    n = int(pts.shape[0])
    if _is_torch(pts):
        import torch
        idx = torch.empty((n, k), dtype=torch.int32, device=pts.device)
        w = torch.empty((n, k), dtype=torch.float32, device=pts.device)
    else:
        idx, w = np.zeros((n, k), np.int32), np.zeros((n, k), np.float32)
    _check(ctx, _lib.mis_skin(ctx, _mem_of(pts), n, _ptr(pts, np.float32), _ptr(idx), _ptr(w)))
    return idx, w


def mis_dbg_set_nodes(ctx, Rt):
    _check(ctx, _lib.mis_dbg_set_nodes(ctx, _mem_of(Rt), _ptr(Rt, np.float32)))


def mis_dbg_frame(ctx, H, W):
    out = np.zeros((H, W, 4), np.float32)
    _check(ctx, _lib.mis_dbg_frame(ctx, MIS_MEM_HOST, _ptr(out)))
    return out


def mis_dbg_associate(ctx, n):
    pix = np.zeros(n, np.int32)
    why = np.zeros(n, np.uint8)
    _check(ctx, _lib.mis_dbg_associate(ctx, MIS_MEM_HOST, _ptr(pix), _ptr(why)))
    return pix, why


def mis_dbg_system(ctx, m, block=6):
    nnz = C.c_int64()
    _check(ctx, _lib.mis_dbg_system(ctx, None, None, None, None, None, C.byref(nnz)))
    nz = nnz.value
    row_ptr = np.zeros(m + 1, np.int32)
    col = np.zeros(nz, np.int32)
    val = np.zeros((nz, block, block), np.float32)
    rhs = np.zeros(block * m, np.float32)
    E = np.zeros(5, np.float64)
    _check(ctx, _lib.mis_dbg_system(ctx, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(rhs), _ptr(E), C.byref(nnz)))
    return dict(row_ptr=row_ptr, col=col, val=val, rhs=rhs, energy=E, nnzb=nz)


def mis_dbg_fuse_register(ctx, H, W, n):
    owner = np.zeros(H * W, np.int64)
    why = np.zeros(n, np.uint8)
    _check(ctx, _lib.mis_dbg_fuse_register(ctx, _ptr(owner), _ptr(why)))
    return owner, why


def mis_prof_name(cat):
    return _lib.mis_prof_name(cat).decode()


def mis_prof_enable(ctx, on=True, light=False):
    """on: event pairs around every kernel group; light: only the K3 and solver groups."""
    _check(ctx, _lib.mis_prof_enable(ctx, (2 if light else 1) if on else 0))


def mis_prof_read(ctx, reset=False):
    ms = np.zeros(MIS_PROF_NCAT, np.float64)
    n = np.zeros(MIS_PROF_NCAT, np.int64)
    _check(ctx, _lib.mis_prof_read(ctx, _ptr(ms), _ptr(n), 1 if reset else 0))
    return {mis_prof_name(i): (float(ms[i]), int(n[i])) for i in range(MIS_PROF_NCAT)}


def mis_launch_count():
    return int(_lib.mis_launch_count())


def mis_dbg_solver_phases(ctx):
    """Microseconds spent in the phases of the last cluster-PCG launch."""
    t = np.zeros(256, np.uint64)
    _check(ctx, _lib.mis_dbg_solver_phases(ctx, _ptr(t)))
    t = t.astype(np.int64).reshape(16, 16)
    t = t[t[:, 0] > 0]
    it1 = None
    if len(t) and (t[:, 14] > 0).all():
        it1 = {}
        if (t[:, 15] == 1).all():   # pipelined PCG
            parts = [("dots_Mw", 8, 9), ("replicate", 9, 10), ("publish", 10, 11), ("cluster_sync", 11, 12),
                     ("scalars", 12, 6), ("spmv", 6, 13), ("update", 13, 14)]
        else:
            parts = [("spmv", 8, 9), ("pAp_sum", 9, 10), ("syncB", 10, 11), ("xr_z", 11, 12),
                     ("replicate_sum", 12, 13), ("syncA", 13, 14)]
        for n, a_, b_ in parts:
            d = (t[:, b_] - t[:, a_]) / 1e3
            it1[n] = (round(float(d.min()), 2), round(float(d.max()), 2))
    if len(t) == 0:
        return {}
    t0 = t[:, 0].min()
    names = ["build_system", "precond", "init", "pcg", "update"]
    out = {}
    for i, n in enumerate(names):
        d = (t[:, i + 1] - t[:, i]) / 1e3
        out[n] = round(float(d.max()), 2)
        out[n + "_min_cta"] = round(float(d.min()), 2)
    out["precond_done_spread"] = round(float((t[:, 2].max() - t[:, 2].min()) / 1e3), 2)
    out["build_done_spread"] = round(float((t[:, 1].max() - t[:, 1].min()) / 1e3), 2)
    out["start_spread"] = round(float((t[:, 0].max() - t0) / 1e3), 2)
    out["total"] = round(float((t[:, 5].max() - t0) / 1e3), 2)
    if it1:
        out["pcg_iteration_1_us_min_max"] = it1
    return out


class Context:
    """Owns one mis_ctx; thin convenience wrapper over the functions above."""

    def __init__(self, params: mis_params | None = None, device=0, stream=None, rank=0, world=1, nccl_id=None):
        self.params = params or mis_default_params()
        self.ptr = mis_create(self.params, device, stream, rank, world, nccl_id)

    def close(self):
        if self.ptr:
            mis_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
