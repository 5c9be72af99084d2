"""Dev: run one dependency level of n isolated windows (F = 64 unless F/B
given) a few times -- the target of ncu captures of the narrow-level kernels.
usage: [WINDOWS=1] [B=4 F=64] python tools/lone_window.py fp32|fp64"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth

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
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
p = P.FseParams(d=14, iterations=100, block_size=B, fft_size=F)
plan = P.build_plan(mask, p)
src = torch.from_numpy(img0).cuda().to(torch.float32 if prec == "fp32" else torch.float64)
m = torch.from_numpy(mask).cuda()
mo = torch.empty_like(m)
for rep in range(4):
    work = src.clone()
    P.run_frames_device([plan], [work], [m], [mo], p, prec)
torch.cuda.synchronize()
print("ok")
