"""Per-CUDA-source-line warp-stall samples and instructions of one ncu report.

usage: python tools/ncu_lines.py REPORT.ncu-rep [min_pct]
Prints the lines above min_pct of all samples, plus the split between the
per-iteration loop (instructions executed >= 90x per warp) and the rest.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_pct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
start = rows.index(hdr) + 1
lines, sass = [], []
for r in rows[start:]:
    if len(r) <= ii:
        continue
    if r[0] and r[2] == "-":
        try:
            lines.append((int(r[si] or 0), int(float(r[ii] or 0)), int(r[0]), r[1].strip()[:100]))
        except ValueError:
            pass
    elif not r[0] and r[3].strip() and r[4] not in ("-", ""):
        try:
            sass.append((int(r[si] or 0), int(float(r[ii] or 0)), int(r[2], 16)))
        except ValueError:
            pass
tot = sum(s for s, *_ in lines) or 1
warps = min(sass, key=lambda x: x[2])[1] if sass else 1  # the entry instruction runs once per warp
print(f"samples {tot}  warps {warps}")
loop = [(s, n) for s, n, _ in sass if n >= 90 * warps]
rest = [(s, n) for s, n, _ in sass if n < 90 * warps]
for name, grp in (("loop", loop), ("setup/other", rest)):
    print(f"{name:12s} samples {100 * sum(s for s, _ in grp) / tot:5.1f}%  inst/warp {sum(n for _, n in grp) / warps:9.1f}")
for s, n, ln, src in sorted(lines, key=lambda x: x[2]):
    if s >= tot * min_pct / 100:
        print(f"{ln:4d} {100 * s / tot:5.1f}%  inst/warp {n / warps:8.1f}  {src}")
