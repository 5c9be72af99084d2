"""Shared-memory wavefronts per CUDA source line of one ncu report (--set full,
--import-source on): where the l1tex shared wavefronts (and the bank-conflict
excess) go.  usage: python tools/ncu_smem_lines.py REPORT [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if "L1 Wavefronts Shared" in r)
iw, ix = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive")
isrc = 1
lines = []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= iw or not (r[0] and r[2] == "-"):  # CUDA source rows (SASS rows have an address)
        continue
    try:
        w, x = float(r[iw] or 0), float(r[ix] or 0)
    except ValueError:
        continue
    if w:
        lines.append((w, x, r[0], r[isrc].strip()[:90]))
tot = sum(w for w, *_ in lines)
totx = sum(x for _, x, *_ in lines)
print(f"shared wavefronts {tot:.0f} (excessive {totx:.0f}, {100 * totx / max(tot, 1):.1f}%)")
for w, x, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{ln:>5} {100 * w / tot:5.1f}%  excess {100 * x / max(w, 1):5.1f}%  {src}")
