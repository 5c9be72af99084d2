"""Dev: device time of ONE dependency level holding n independent windows
(n = 1, 148, 2*148, ...), per FFT size and precision -- the per-level cost
the strip-sharding scaling model needs (tools/scaling_model.py).

Windows are isolated 4x4 blocks (B = F/16, d = 14) far apart on a synthetic
frame, so the plan is a single level of exactly n windows.  Prints one JSON
line per (F, precision, n) with the kernel time of that level (fse timing).
"""
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
SMS = torch.cuda.get_device_properties(0).multi_processor_count
img0, _ = synth.config_scene(5)  # 2160 x 3840
out = []
for B, F in ((2, 32), (4, 64), (8, 128)):
    p = P.FseParams(d=14, iterations=100, block_size=B, fft_size=F)
    R = -(-14 // B)
    step = 2 * R + 2  # blocks apart: windows never overlap, one level
    rows, cols = 2160 // B, 3840 // B
    cand = [(r, c) for r in range(R + 1, rows - R - 1, step) for c in range(R + 1, cols - R - 1, step)]
    for prec in ("fp32", "fp64"):
        if F == 128 and prec == "fp64":
            continue
        for n in (1, SMS, 2 * SMS, 3 * SMS, 4 * SMS, 6 * SMS, 8 * SMS):
            if n > len(cand):
                continue
            mask = np.zeros((2160, 3840), np.uint8)
            for r, c in cand[:n]:
                mask[r * B:(r + 1) * B, c * B:(c + 1) * B] = 1
            plan = P.build_plan(mask, p)
            assert plan.n_levels == 1 and plan.n_processed == n, (plan.n_levels, plan.n_processed, n)
            tdt = torch.float32 if prec == "fp32" else torch.float64
            src = torch.from_numpy(img0).cuda().to(tdt)
            work = torch.empty_like(src)
            m = torch.from_numpy(mask).cuda()
            mo = torch.empty_like(m)
            ts = []
            for rep in range(6):
                work.copy_(src)
                torch.cuda.synchronize()
                L.fse_timing_read(None, None, None)
                L.fse_timing_enable(1)
                P.run_frames_device([plan], [work], [m], [mo], p, prec)
                torch.cuda.synchronize()
                L.fse_timing_enable(0)
                kms = ctypes.c_double()
                L.fse_timing_read(ctypes.byref(kms), None, None)
                if rep >= 2:
                    ts.append(kms.value)
            rec = {"F": F, "B": B, "precision": prec, "windows": n, "windows_per_sm": n / SMS,
                   "level_ms": float(np.median(ts))}
            out.append(rec)
            print(json.dumps(rec), flush=True)
