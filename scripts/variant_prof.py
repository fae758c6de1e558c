"""Per-kernel-group breakdown (mis_prof) of the bench step for a flag variant.
    python scripts/variant_prof.py [config] [flag ...]   flags: joint affine lm grid"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1803_02009_b200 import mis as M
cfgn = sys.argv[1] if len(sys.argv) > 1 else "c3"
names = sys.argv[2:]
F = {"joint": M.MIS_F_JOINT_POSE, "affine": M.MIS_F_AFFINE, "lm": M.MIS_F_LM, "grid": M.MIS_F_GRID_SOLVER}
dev = torch.device("cuda", 0)
sc = bench.load_workload(cfgn, 0); cfg = sc["cfg"]; it = sc["intr"]
intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
td = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
s0 = torch.cuda.current_stream()
ctx = M.Context(bench.params_for(cfg, M), stream=s0.cuda_stream)
n = sc["xyz"].shape[0]; cap = n + cfg.H * cfg.W + 16
M.mis_set_model(ctx.ptr, td(sc["xyz"]), td(sc["nrm"]), td(sc["rgb"]), td(sc["weight"]), td(sc["stamp"]), capacity=cap)
M.mis_set_graph(ctx.ptr, td(sc["g"]), td(sc["nbr"]))
st = M.mis_get_model(ctx.ptr, cfg.k, device=True)
ctx.close()
pv = bench.params_for(cfg, M)
for nm in names:
    pv.flags |= F[nm]
cv = M.Context(pv, stream=s0.cuda_stream)
g_d, nbr_d, depth_d, rgb_d = td(sc["g"]), td(sc["nbr"]), td(sc["depth"]), td(sc["rgb_obs"])
fs_d, fd_d = td(sc["feat_src"]), td(sc["feat_dst"])
def step():
    M.mis_set_model(cv.ptr, st["xyz"], st["nrm"], st["rgb"], st["weight"], st["stamp"], st["ids"], capacity=cap)
    M.mis_set_graph(cv.ptr, g_d, nbr_d, st["knn_idx"], st["knn_w"])
    M.mis_register(cv.ptr, depth_d, intr, sc["pose"], fs_d, fd_d, report=False)
    M.mis_warp(cv.ptr)
    M.mis_fuse(cv.ptr, rgb_d, 1)
for _ in range(3):
    step()
torch.cuda.synchronize()
K = 10
M.mis_prof_read(cv.ptr, reset=True)
M.mis_prof_enable(cv.ptr, True)
for _ in range(K):
    step()
torch.cuda.synchronize()
M.mis_prof_enable(cv.ptr, False)
pr = M.mis_prof_read(cv.ptr, reset=True)
print(cfgn, names, {k: round(v[0] / K, 4) for k, v in pr.items() if v[0] > 0}, "sum", round(sum(v[0] for v in pr.values()) / K, 4))
