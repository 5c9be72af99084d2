"""Dev: where a lone window's latency goes -- device time of one level of n
isolated F=64 windows (n = 1 and one per SM) against the iteration count
(I = 0, 1, 10, 50, 100): the intercept is the set-up (staging, DFT passes, W
plane, write-back) plus launch, the slope the per-iteration cost.
Run once per kernel variant (FSE_F64L=12/22 select the wide fp64 variants).
usage: python tools/latency_breakdown.py [fp32|fp64]...
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
img0, _ = synth.config_scene(5)
B, F = 4, 64
precs = sys.argv[1:] or ["fp32", "fp64"]
R = -(-14 // B)
step = 2 * R + 2
rows, cols = 2160 // B, 3840 // B
cand = [(r, c) for r in range(R + 1, rows - R - 1, step) for c in range(R + 1, cols - R - 1, step)]
for prec in precs:
    for n in (1, SMS):
        mask = np.zeros((2160, 3840), np.uint8)
        for r, c in cand[:n]:
            mask[r * B:(r + 1) * B, c * B:(c + 1) * B] = 1
        for I in (0, 1, 10, 50, 100):
            p = P.FseParams(d=14, iterations=I, block_size=B, fft_size=F)
            plan = P.build_plan(mask, p)
            tdt = torch.float32 if prec == "fp32" else torch.float64
            src = torch.from_numpy(img0).cuda().to(tdt)
            work = torch.empty_like(src)
            m = torch.from_numpy(mask).cuda()
            mo = torch.empty_like(m)
            ts = []
            for rep in range(8):
                work.copy_(src)
                torch.cuda.synchronize()
                L.fse_timing_read(None, None, None)
                L.fse_timing_enable(1)
                P.run_frames_device([plan], [work], [m], [mo], p, prec)
                torch.cuda.synchronize()
                L.fse_timing_enable(0)
                kms = ctypes.c_double()
                L.fse_timing_read(ctypes.byref(kms), None, None)
                if rep >= 3:
                    ts.append(kms.value)
            print(json.dumps({"variant": os.environ.get("FSE_F64L", "0"), "precision": prec, "windows": n,
                              "iterations": I, "level_us": 1e3 * float(np.median(ts))}), flush=True)
