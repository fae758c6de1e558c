"""GPU timeline of one bench step (torch.profiler / CUPTI): every kernel and copy with its
start, duration and the idle gap before it, so host-bound stretches show up.

    python scripts/timeline.py [--config c3] [--steps 3] [--top 0]
"""
import argparse
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_1803_02009_b200 import mis as M

    dev = torch.device("cuda", 0)
    sc = bench.load_workload(args.config, 0)
    cfg = sc["cfg"]
    it = sc["intr"]
    intr = M.intrinsics(it["fx"], it["fy"], it["cx"], it["cy"], it["W"], it["H"])
    stream = torch.cuda.current_stream()
    td = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctx = M.Context(bench.params_for(cfg, M), stream=stream.cuda_stream)
    n = sc["xyz"].shape[0]
    cap = n + cfg.H * cfg.W + 16
    M.mis_set_model(ctx.ptr, td(sc["xyz"]), td(sc["nrm"]), td(sc["rgb"]), td(sc["weight"]), td(sc["stamp"]),
                    capacity=cap)
    M.mis_set_graph(ctx.ptr, td(sc["g"]), td(sc["nbr"]))
    st = M.mis_get_model(ctx.ptr, cfg.k, device=True)
    g_d, nbr_d = td(sc["g"]), td(sc["nbr"])
    depth_d, rgb_d = td(sc["depth"]), td(sc["rgb_obs"])
    fs_d, fd_d = td(sc["feat_src"]), td(sc["feat_dst"])

    def step():
        M.mis_set_model(ctx.ptr, st["xyz"], st["nrm"], st["rgb"], st["weight"], st["stamp"], st["ids"], capacity=cap)
        M.mis_set_graph(ctx.ptr, g_d, nbr_d, st["knn_idx"], st["knn_w"])
        M.mis_register(ctx.ptr, depth_d, intr, sc["pose"], fs_d, fd_d, report=False)
        M.mis_warp(ctx.ptr)
        return M.mis_fuse(ctx.ptr, rgb_d, 1)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
    fn = os.path.join(tempfile.gettempdir(), "mis_trace.json")
    prof.export_chrome_trace(fn)
    ev = json.load(open(fn))["traceEvents"]
    gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    gpu.sort(key=lambda e: e["ts"])
    # the last step: from the last k_load_model
    starts = [i for i, e in enumerate(gpu) if "k_load_model" in e["name"]]
    s0 = starts[-1]
    seq = gpu[s0:]
    t0 = seq[0]["ts"]
    busy = sum(e["dur"] for e in seq)
    end = max(e["ts"] + e["dur"] for e in seq)
    print(f"step span {end - t0:.1f} us, busy {busy:.1f} us, idle {end - t0 - busy:.1f} us, {len(seq)} ops")
    prev_end = t0
    for e in seq:
        gap = e["ts"] - prev_end
        name = e["name"].split("(")[0].replace("void ", "").replace("mis::", "")[:60]
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} gap {gap:7.1f}  {name}")
        prev_end = max(prev_end, e["ts"] + e["dur"])


if __name__ == "__main__":
    main()
