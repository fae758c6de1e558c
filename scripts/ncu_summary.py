"""Summarise an ncu launch list + full capture into profiles/.

    python scripts/ncu_summary.py <tag> [--round r2] [--config c3]

Reads gpurun_out/launches_<tag>.csv and gpurun_out/full_<tag>.ncu-rep and writes
profiles/<round>_launches_<config>.csv (per-kernel aggregate), profiles/<round>_ncu_summary_<config>.md
and profiles/<round>_traffic_<config>.json (DRAM bytes per launch of each captured kernel group,
averaged over the captured launches; read by bench.py --config <config> for the roofline "traffic").
"""
import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GROUP = {"k_assoc_points": "assoc_points", "k_assoc_chunks": "assoc_points", "k_accum_points": "accum_points", "k_pcg_cluster": "solve", "k_solve": "solve",
         "k_finalize": "finalize", "k_assemble_graph": "assemble_graph", "k_frame_prep": "frame_prep",
         "k_warp_model": "warp_model", "k_fuse_register": "fuse_register", "k_fuse_apply": "fuse_apply"}


def short(name):
    n = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    n = n.split("(")[0]
    n = n.replace("void ", "").replace("mis::", "")
    return n


def launches(tag):
    rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv"))))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        n = short(r[ki])
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(n, [0.0, 0])
        a[0] += v
        a[1] += 1
    return agg


def full(tag):
    rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}.ncu-rep")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    keys = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read",
            "dram__bytes_write.sum": "dram_write", "launch__registers_per_thread": "regs",
            "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
            "smsp__inst_executed.sum": "warp_instructions", "lts__t_bytes.sum": "l2_bytes",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
            "launch__grid_size": "grid", "launch__block_size": "block"}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
             "ns": 1e-3, "us": 1, "ms": 1e3}
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, nm in keys.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[nm] = v * scale.get(units[i], 1)
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(r[i]), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        d["top_stalls"] = [(k, round(100 * v / tot, 1)) for v, k in sorted(st, reverse=True)[:5]]
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--round", default="r2")
    ap.add_argument("--config", default="c3")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    agg = launches(a.tag)
    total = sum(v[0] for v in agg.values())
    with open(os.path.join(ROOT, "profiles", f"{a.round}_launches_{a.config}.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_us", "avg_us", "share_pct"])
        for n, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
            w.writerow([n, c, round(v / 1e3, 2), round(v / c / 1e3, 3), round(100 * v / total, 2)])
    fl = full(a.tag)
    traffic = {}
    lines = [f"# ncu summary ({a.round}, bench --config {a.config}, capture tag {a.tag})", "",
             "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1` (cold-cache, serialised: "
             "shares, not absolute times). Full capture: `ncu --set full --clock-control none --import-source on`.",
             "", "## Launch list (top 15 by total time)", "", "| kernel | launches | avg us | share % |", "|---|---|---|---|"]
    for n, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:15]:
        lines.append(f"| {n} | {c} | {v / c / 1e3:.2f} | {100 * v / total:.1f} |")
    lines += ["", "## Full captures", "",
              "| kernel | us | DRAM read MB | DRAM write MB | L2 MB | regs | occ % | SM thr % | top stalls |",
              "|---|---|---|---|---|---|---|---|---|"]
    for d in fl:
        lines.append(f"| {d['kernel']} | {d.get('duration', 0):.1f} | {d.get('dram_read', 0) / 1e6:.2f} | "
                     f"{d.get('dram_write', 0) / 1e6:.2f} | {d.get('l2_bytes', 0) / 1e6:.1f} | {d.get('regs', 0):.0f} | "
                     f"{d.get('achieved_occupancy_pct', 0):.1f} | {d.get('sm_throughput_pct', 0):.1f} | {d['top_stalls']} |")
        g = next((v for k, v in GROUP.items() if d["kernel"].startswith(k)), None)
        if g:
            traffic.setdefault(g, []).append(d.get("dram_read", 0) + d.get("dram_write", 0))
    open(os.path.join(ROOT, "profiles", f"{a.round}_ncu_summary_{a.config}.md"), "w").write("\n".join(lines) + "\n")
    json.dump({"config": a.config, "source": f"gpurun_out/full_{a.tag}.ncu-rep (ncu --set full, dram__bytes_read.sum "
                                             "+ dram__bytes_write.sum, mean over the captured launches)",
               "bytes_per_launch": {g: int(sum(v) / len(v)) for g, v in traffic.items()},
               "launches_captured": {g: len(v) for g, v in traffic.items()}},
              open(os.path.join(ROOT, "profiles", f"{a.round}_traffic_{a.config}.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
