"""Static instruction mix of the fast kernel's per-iteration loop (cuobjdump SASS).

usage: python tools/sass_loop.py [float|double] [F] [print]
The loop is the block between the back-edge BRA that follows the first CREDUX
and its target.
"""
import re
import subprocess
import sys
from collections import Counter

ty = sys.argv[1] if len(sys.argv) > 1 else "float"
F = sys.argv[2] if len(sys.argv) > 2 else "64"
show = len(sys.argv) > 3
sass = subprocess.run(["cuobjdump", "-sass", "paper_2207_00233_b200/libfse_b200.so"],
                      capture_output=True, text=True).stdout
tag = {"float": "If", "double": "Id"}[ty] + "Li" + F
for f in re.split(r"\n\s+Function : ", sass)[1:]:
    name = f.split("\n")[0]
    if "15fse_fast_kernel" not in name or tag not in name or "Li0ELb0E" not in name:
        continue
    ins = []
    for l in f.split("\n"):
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    first = next(i for i, (_, s) in enumerate(ins) if "CREDUX" in s)
    for i in range(first, len(ins)):
        m = re.match(r"(@!?U?P\d\s+)?BRA(\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", ins[i][1])
        if m and int(m.group(3), 16) <= ins[first][0]:
            start = next(k for k, (a, _) in enumerate(ins) if a == int(m.group(3), 16))
            body = ins[start:i + 1]
            break
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0] for _, s in body)
    print(f"{name[:70]}: loop {len(body)} instructions")
    print("  " + ", ".join(f"{k} {v}" for k, v in ops.most_common()))
    if show:
        for a, s in body:
            print(f"  {a:6x} {s}")
