"""Static instruction mix of the fast kernel's per-iteration loop (cuobjdump SASS).

usage: python tools/sass_loop.py [float|double] [F] [print] [lib.so]
The loop is the smallest back-edge region that contains a CREDUX and FFMA2/DFMA
work (the per-iteration argmax plus the spectrum update)."""
import collections
import re
import subprocess
import sys

ty = sys.argv[1] if len(sys.argv) > 1 else "float"
F = sys.argv[2] if len(sys.argv) > 2 else "64"
show = len(sys.argv) > 3 and sys.argv[3] == "print"
lib = sys.argv[4] if len(sys.argv) > 4 else "paper_2207_00233_b200/libfse_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
tag = {"float": "If", "double": "Id"}[ty] + "Li" + F
work = "FFMA2" if ty == "float" else "DFMA"
for f in re.split(r"\n\s+Function : ", sass)[1:]:
    name = f.split("\n")[0]
    if "15fse_fast_kernel" not in name or tag not in name or not re.search(r"EEELi0ELb0E(Lb[01]E)?EEv", name):
        continue
    ins = []
    for line in f.split("\n"):
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    best = None
    for a, t in ins:
        m = re.match(r"(@!?U?P\w+\s+)?BRA(\.\w+)?\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", t)
        if m and int(m.group(3), 16) < a:
            body = [x for x in ins if int(m.group(3), 16) <= x[0] <= a]
            if any("CREDUX" in x[1] for x in body) and any(work in x[1] for x in body):
                if best is None or len(body) < len(best):
                    best = body
    if not best:
        continue
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for _, t in best)
    print(f"{name[:90]}: loop {len(best)} instructions")
    print("  " + ", ".join(f"{k} {v}" for k, v in ops.most_common()))
    if show:
        for a, t in best:
            print(f"  {a:6x} {t}")
