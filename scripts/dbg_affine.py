"""Debug: repeated affine registrations on one context (bench-like), status and energies per step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1803_02009_b200 import mis as M
cfgn = sys.argv[1] if len(sys.argv) > 1 else "c3"
flag = int(sys.argv[2]) if len(sys.argv) > 2 else M.MIS_F_AFFINE
dev = torch.device("cuda", 0)
sc = bench.load_workload(cfgn, 0); cfg = sc["cfg"]; it = sc["intr"]
intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
td = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
st0 = torch.cuda.current_stream()
ctx = M.Context(bench.params_for(cfg, M), stream=st0.cuda_stream)
n = sc["xyz"].shape[0]; cap = n + cfg.H * cfg.W + 16
M.mis_set_model(ctx.ptr, td(sc["xyz"]), td(sc["nrm"]), td(sc["rgb"]), td(sc["weight"]), td(sc["stamp"]), capacity=cap)
M.mis_set_graph(ctx.ptr, td(sc["g"]), td(sc["nbr"]))
st = M.mis_get_model(ctx.ptr, cfg.k, device=True)
ctx.close()
pv = bench.params_for(cfg, M); pv.flags |= flag
cv = M.Context(pv, stream=st0.cuda_stream)
g_d, nbr_d, depth_d, rgb_d = td(sc["g"]), td(sc["nbr"]), td(sc["depth"]), td(sc["rgb_obs"])
fs_d, fd_d = td(sc["feat_src"]), td(sc["feat_dst"])
for k in range(8):
    M.mis_set_model(cv.ptr, st["xyz"], st["nrm"], st["rgb"], st["weight"], st["stamp"], st["ids"], capacity=cap)
    M.mis_set_graph(cv.ptr, g_d, nbr_d, st["knn_idx"], st["knn_w"])
    try:
        rep = M.report_dict(M.mis_register(cv.ptr, depth_d, intr, sc["pose"], fs_d, fd_d, report=True))
        print(k, "ok", rep["energy"][:, 4], rep["pcg_rel_res"])
    except M.MisError as e:
        print(k, "ERR", e)
    M.mis_warp(cv.ptr)
    M.mis_fuse(cv.ptr, rgb_d, 1)
