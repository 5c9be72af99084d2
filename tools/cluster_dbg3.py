import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2207_00233_b200 as P
H, W = 40, 44
rng = np.random.default_rng(1)
img = rng.uniform(0, 255, (H, W)).round()
mask = np.zeros((H, W), np.uint8)
mask[2:6, 2:6] = 1  # a clipped-window block near the corner
p = P.FseParams(d=14, iterations=int(sys.argv[1]), block_size=4, fft_size=64)
out, om, rep = P.conceal(img, mask, p, precision="fp32")
print("ok", rep.blocks_processed)
