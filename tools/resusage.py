"""Per-kernel registers / stack / local memory of the built library (cuobjdump)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2207_00233_b200/libfse_b200.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "fse_fast"
out = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True).stdout
name = None
for line in out.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:\d+ LOCAL:(\d+)", line)
    if m and name and pat in name:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = dem.replace("fse::", "").replace("(FastArgs, FastLayout)", "")
        print(f"REG {m.group(1):>3} STACK {m.group(2):>3} LOCAL {m.group(3):>3}  {dem}")
