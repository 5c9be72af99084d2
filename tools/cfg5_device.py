"""Dev: device time of the config-5 4K frame (plan prebuilt, whole frame on one
GPU, level launches) for the given block sizes and precision.
usage: python tools/cfg5_device.py fp64 2 8"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
img, mask = synth.config_scene(5)
for B in [int(x) for x in sys.argv[2:]] or [2, 4, 8]:
    F = {2: 32, 4: 64, 8: 128}[B]
    p = P.FseParams(d=14, iterations=100, block_size=B, fft_size=F)
    plan = P.build_plan(mask, p)
    src = torch.from_numpy(img).cuda().to(torch.float32 if prec == "fp32" else torch.float64)
    work = torch.empty_like(src)
    m = torch.from_numpy(mask).cuda()
    mo = torch.empty_like(m)
    ts = []
    for rep in range(4):
        work.copy_(src)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        P.run_frames_device([plan], [work], [m], [mo], p, prec)
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1))
    print(f"{os.environ.get('TAGV', 'main')} B={B} {prec}: {np.median(ts):.2f} ms ({plan.n_levels} levels)", flush=True)
