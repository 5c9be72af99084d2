"""Dev: sustained throughput of ConcealStream on config-4 frames (frames pushed
one by one from host memory, results read back) vs conceal_batch calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth
from concurrent.futures import ThreadPoolExecutor

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
with ThreadPoolExecutor(16) as ex:
    sc = list(ex.map(lambda f: synth.config_scene(4, f), range(n)))
imgs = [s[0] for s in sc]; msks = [s[1] for s in sc]
p = P.FseParams(d=14, iterations=100, block_size=4, fft_size=64)
for batch in (8, 16, 32):
    with P.ConcealStream(p, imgs[0].shape, batch=batch, depth=3) as st:
        for rep, loops in ((0, 1), (1, 1), (2, 4)):  # the last: 4 x n frames in one stream (sustained)
            t = time.perf_counter(); got = 0
            for f in range(n * loops):
                got += len(st.push(imgs[f % n], msks[f % n]))
            got += len(st.flush())
            dt = time.perf_counter() - t
            print(f"stream batch {batch:2d} rep {rep}: {n * loops} frames in {1e3*dt:.1f} ms = {1e3*dt/(n * loops):.2f} ms/frame ({got} back)", flush=True)
ih = torch.from_numpy(np.stack(imgs)).pin_memory(); mh = torch.from_numpy(np.stack(msks)).pin_memory()
oi = torch.empty(ih.shape, dtype=torch.float64, pin_memory=True)  # conceal_batch defaults to fp64
om = torch.empty(mh.shape, dtype=torch.uint8, pin_memory=True)
for rep in range(3):
    t = time.perf_counter()
    P.conceal_batch(ih, mh, p, out_images=oi, out_masks=om, reports=False)
    dt = time.perf_counter() - t
    print(f"conceal_batch({n}) rep {rep}: {1e3*dt:.1f} ms = {1e3*dt/n:.2f} ms/frame", flush=True)
