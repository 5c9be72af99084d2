"""Dev: host plan time of the config-5 4K frame (B = 2 / 4 / 8) against the
plan thread count (fse_plan_build_threads), checking that every thread count
gives the same plan.  FSE_PLAN_TIMING=1 adds the stage breakdown.
usage: python tools/plan_threads_time.py [threads ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import synth
from paper_2207_00233_b200.conceal import build_plan

img, mask = synth.config_scene(5)
threads = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8, 16]
print("usable cpus", len(os.sched_getaffinity(0)), flush=True)
for B, F in ((2, 32), (4, 64), (8, 128)):
    p = P.FseParams(d=14, iterations=100, block_size=B, fft_size=F)
    ref = None
    for T in threads + [0]:
        ts = []
        for r in range(4):
            t = time.perf_counter()
            pl = build_plan(mask, p, plan_threads=T)
            ts.append(time.perf_counter() - t)
        s = (pl.batches(), pl.levels(), pl.ranks().tolist())
        if ref is None:
            ref = s
        print(f"B={B} threads={T or 'auto'}: {1e3 * min(ts):.1f} ms (median {1e3 * np.median(ts):.1f}) "
              f"same={s == ref}", flush=True)
