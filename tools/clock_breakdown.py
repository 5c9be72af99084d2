"""Dev: clock64 phase breakdown of a lone window (CTA 0, thread 0) on the
instrumented build:
    FSE_BUILD_TAG=clk FSE_NVCC_DEFS=-DFSE_CLOCKS python -m paper_2207_00233_b200.build
    FSE_LIB=paper_2207_00233_b200/variants/libfse_b200_clk.so python tools/clock_breakdown.py fp64
Prints set-up phases and the per-iteration split (argmax+barrier, decode,
update loop) in SM cycles, median over iterations 10..89."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import _lib, synth

L = _lib.lib()
L.fse_debug_clocks.argtypes = [ctypes.c_void_p, ctypes.c_int]
img0, _ = synth.config_scene(5)
B, F = int(os.environ.get("B", 4)), int(os.environ.get("F", 64))
n = int(os.environ.get("WINDOWS", 1))
R = -(-14 // B)
step = 2 * R + 2
rows, cols = 2160 // B, 3840 // B
cand = [(r, c) for r in range(R + 1, rows - R - 1, step) for c in range(R + 1, cols - R - 1, step)]
mask = np.zeros((2160, 3840), np.uint8)
for r, c in cand[:n]:
    mask[r * B:(r + 1) * B, c * B:(c + 1) * B] = 1
for prec in sys.argv[1:] or ["fp32", "fp64"]:
    p = P.FseParams(d=14, iterations=100, block_size=B, fft_size=F)
    plan = P.build_plan(mask, p)
    tdt = torch.float32 if prec == "fp32" else torch.float64
    src = torch.from_numpy(img0).cuda().to(tdt)
    m = torch.from_numpy(mask).cuda()
    mo = torch.empty_like(m)
    for rep in range(3):
        work = src.clone()
        P.run_frames_device([plan], [work], [m], [mo], p, prec)
        torch.cuda.synchronize()
    clk = np.zeros(1032, np.int64)
    assert L.fse_debug_clocks(clk.ctypes.data, 1032) == 0
    c = clk
    it = np.array([c[8 + 4 * i: 12 + 4 * i] for i in range(100)])
    nxt = np.append(it[1:, 0], c[5])
    seg = {"argmax+barrier": np.median(it[10:90, 1] - it[10:90, 0]),
           "decode": np.median(it[10:90, 2] - it[10:90, 1]),
           "update loop": np.median(nxt[10:90] - it[10:90, 2])}
    rec = {"precision": prec, "F": F, "windows": n, "variant": os.environ.get("FSE_F64L", "0"),
           "setup_cycles": {"twiddles+staging": int(c[1] - c[0]), "column pass": int(c[2] - c[1]),
                            "x row pass": int(c[3] - c[2]), "w row pass + W plane": int(c[4] - c[3]),
                            "(w partials)": int(c[1000] - c[3]), "(w combine)": int(c[1001] - c[1000]),
                            "(W mirror rows)": int(c[4] - c[1001])},
           "loop_cycles": int(c[5] - c[4]), "writeback_cycles": int(c[6] - c[5]),
           "per_iteration_cycles": {k: float(v) for k, v in seg.items()}}
    print(json.dumps(rec), flush=True)
