"""Run the bench's Alg. 2 sequence (register -> warp -> fuse -> filter -> regenerate) of a config and check
the model after every stage of every frame: non-finite positions, bounding box, sizes, registration energies.
    python scripts/dbg_seq.py c4 100"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1803_02009_b200 import mis as M  # noqa: E402
from paper_1803_02009_b200 import synth  # noqa: E402
import bench  # noqa: E402

cfgname, nfr = sys.argv[1], int(sys.argv[2])
dev = torch.device("cuda", 0)
sc = bench.load_workload(cfgname, 0)
cfg, it = sc["cfg"], sc["intr"]
intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
td = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
base, frames = synth.make_sequence_frames(cfgname, nfr)
n0, m0 = base["xyz"].shape[0], base["g"].shape[0]
ext = base["xyz"].max(0) - base["xyz"].min(0)
box = float(np.sqrt(ext[0] * ext[1] / n0))
node = 1.3 * float(np.sqrt(ext[0] * ext[1] / m0))
ef = td(np.zeros((0, 3), np.float32))
cs = M.Context(bench.params_for(cfg, M), device=0, stream=torch.cuda.current_stream().cuda_stream)
M.mis_set_model(cs.ptr, td(base["xyz"]), td(base["nrm"]), td(base["rgb"]), td(base["weight"]), td(base["stamp"]),
                capacity=n0 + 4 * cfg.H * cfg.W)
M.mis_set_graph(cs.ptr, td(base["g"]), td(base["nbr"]))
print("box", box, "node grid", node, "n0", n0, "m0", m0)


def check(tag, fi):
    mod = M.mis_get_model(cs.ptr, cfg.k)
    x = mod["xyz"]
    fin = np.isfinite(x).all(1)
    lo, hi = x[fin].min(0), x[fin].max(0)
    bad = (~fin).sum()
    span = (hi - lo) / box
    if bad or (span > 2 ** 20).any():
        print(f"frame {fi} after {tag}: n {x.shape[0]} non-finite {bad} lo {lo} hi {hi} span/box {span}")
        return False
    return True


for q, f in enumerate(frames):
    fi = f["frame"]
    rep = M.report_dict(M.mis_register(cs.ptr, td(f["depth"]), intr, f["pose"], ef, ef))
    M.mis_warp(cs.ptr)
    if not check("warp", fi):
        print("energies", rep["energy"][:, 4], "n_assoc", rep["n_assoc"])
        Rt = M.mis_get_nodes_f64(cs.ptr, M.mis_get_graph_size(cs.ptr) if hasattr(M, "mis_get_graph_size") else 0)
        break
    n_f, _ = M.mis_fuse(cs.ptr, td(f["rgb_obs"]), fi)
    if not check("fuse", fi):
        print("energies", rep["energy"][:cfg.gn_iters, 4], "n_assoc", rep["n_assoc"][:cfg.gn_iters])
        print("E parts last", rep["energy"][cfg.gn_iters - 1])
        mm = M.mis_get_model(cs.ptr, cfg.k)
        x = mm["xyz"]
        far = np.linalg.norm(x, axis=1) > 1e4
        print("far points", far.sum(), "stamps", np.unique(mm["stamp"][far])[:10], "weights", mm["weight"][far][:5])
        print("their knn", mm["knn_idx"][far][:3], mm["knn_w"][far][:3])
        break
    try:
        n_k, st = M.mis_filter(cs.ptr, box, fi, 10, 3.0)
    except M.MisError as ex:
        print("filter error at frame", fi, ex)
        check("fuse(again)", fi)
        break
    m_k = M.mis_regenerate_nodes(cs.ptr, node)
    if q % 10 == 0:
        print(f"frame {fi}: fused {n_f} kept {n_k} nodes {m_k} E0 {rep['energy'][0, 4]:.4g} E_last {rep['energy'][cfg.gn_iters - 1, 4]:.4g}")
print("done")
