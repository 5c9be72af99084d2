"""Dev: exercise the cluster variants on small cases, one at a time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth
case = sys.argv[1]
img, mask = synth.config_scene(1)
prec, F, B = {"f32_64": ("fp32", 64, 4), "f64_64": ("fp64", 64, 4), "f32_32": ("fp32", 32, 2),
              "f64_32": ("fp64", 32, 2)}[case]
img, mask = img[:64, :64].copy(), mask[:64, :64].copy()
mask[20:36, 20:36] = 1
p = P.FseParams(d=14, iterations=int(sys.argv[2]) if len(sys.argv) > 2 else 10, block_size=B, fft_size=F)
out, om, rep = P.conceal(img, mask, p, precision=prec)
print(case, "ok", rep.blocks_processed, rep.levels)
