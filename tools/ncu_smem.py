"""Per-CUDA-source-line shared-memory wavefronts (and excess from bank
conflicts) of one ncu report, split loop vs setup like ncu_lines.py.

usage: python tools/ncu_smem.py REPORT.ncu-rep [min_pct]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_pct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if "L1 Wavefronts Shared" in r)
wi, xi, ii = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive"), hdr.index(
    "Instructions Executed")
start = rows.index(hdr) + 1
lines, sass = [], []
for r in rows[start:]:
    if len(r) <= wi:
        continue
    try:
        if r[0] and r[2] == "-":
            lines.append((float(r[wi] or 0), float(r[xi] or 0), int(r[0]), r[1].strip()[:90]))
        elif not r[0] and r[3].strip() and r[4] not in ("-", ""):
            sass.append((float(r[wi] or 0), float(r[ii] or 0), int(r[2], 16)))
    except ValueError:
        pass
tot = sum(w for w, *_ in lines) or 1
warps = min(sass, key=lambda x: x[2])[1] if sass else 1
loop = sum(w for w, n, _ in sass if n >= 90 * warps)
print(f"shared wavefronts {tot:.0f}  per warp {tot / warps:.0f}  loop {100 * loop / tot:.1f}%")
for w, x, ln, src in sorted(lines, key=lambda t: t[2]):
    if w >= tot * min_pct / 100:
        print(f"{ln:4d} {100 * w / tot:5.1f}%  excess {100 * x / max(w, 1):4.1f}%  {src}")
