"""Per-CUDA-line summary of an ncu report: python scripts/ncu_lines.py <rep> <kernel-regex> [top]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, hdr, fname = [], None, ""
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 6 and r[0].isdigit() and r[2] == "-":
        rows.append([fname] + r)
si, ii = hdr.index("# Samples") + 1, hdr.index("Instructions Executed") + 1
ts = sum(float(r[si] or 0) for r in rows); ti = sum(float(r[ii] or 0) for r in rows)
print(f"samples {ts:.0f} instructions {ti:.0f}")
for r in sorted(rows, key=lambda r: -float(r[si] or 0))[:top]:
    print(f"{r[0][:14]:>14}:{r[1]:<5} {100*float(r[si])/ts:5.1f}% samp {100*float(r[ii])/ti:5.1f}% inst  {r[2].strip()[:80]}")
