"""Scaling model of config-5 strip sharding, from measured inputs.

usage: python tools/scaling_model.py LATENCY.jsonl [--precision fp32|fp64] [--sync-us 4]

Inputs:
  * LATENCY.jsonl: tools/window_latency.py on a B200 -- the device time of one
    dependency level holding n independent windows, per FFT size/precision;
  * the real config-5 plan (C++ planner, run here): every block's dependency
    level, and the row bands strips.band_partition gives N ranks.
Model (per-level halo protocol, the one implemented): a rank runs level l
after its neighbours finished level l-1, so the step is
    T(N) = sum_l max_r T_lat(n_{l,r}) + L * t_sync(N)
with n_{l,r} the rank's windows of level l and T_lat interpolated from the
measured level times (piecewise linear in n, waves beyond the largest
measured n).  t_sync(1) = 0.  The same sum at N = 1 is checked against the
measured whole-frame device time (tools/bench_configs.py).  Frame-parallel
config 4 has no coupling: T(N) = T(1) * (frames on the busiest rank) / 64.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2207_00233_b200 as P
from paper_2207_00233_b200 import strips, synth


def load(path, prec):
    cal = {}
    for line in open(path):
        if not line.strip().startswith("{"):
            continue
        r = json.loads(line)
        if r["precision"] == prec:
            cal.setdefault(r["F"], []).append((r["windows"], r["level_ms"]))
    return {F: sorted(v) for F, v in cal.items()}


def t_lat(points, n):
    if n <= 0:
        return 0.0
    xs = np.array([p[0] for p in points], float)
    ys = np.array([p[1] for p in points], float)
    if n <= xs[-1]:
        return float(np.interp(n, xs, ys))
    # beyond the largest measured level: extra full waves at the last slope
    slope = (ys[-1] - ys[-2]) / (xs[-1] - xs[-2])
    return float(ys[-1] + slope * (n - xs[-1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("latency")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--sync-us", type=float, default=4.0,
                    help="per-level neighbour flag wait at N > 1 (cuStreamWaitValue32 + signal kernel)")
    a = ap.parse_args()
    cal = load(a.latency, a.precision)
    img, mask = synth.config_scene(5)
    res = {}
    for B, F in ((2, 32), (4, 64), (8, 128)):
        if F not in cal:
            continue
        p = P.FseParams(d=14, iterations=100, block_size=B, fft_size=F)
        plan = P.build_plan(mask, p)
        R = strips.halo_rows(p)
        rows, cols = plan.rows, plan.cols
        levels = plan.levels()
        processed = (plan.ranks() != np.iinfo(np.int32).max).reshape(rows, cols)
        row_of_level = [np.asarray(lv, np.int64) // cols for lv in levels]
        out, lb = {}, {}
        for N in (1, 2, 4, 8):
            bands = strips.band_partition(processed.sum(axis=1), N, R)
            edges = np.array([b[0] for b in bands] + [bands[-1][1]])
            tot = 0.0
            for rl in row_of_level:
                per_rank = np.histogram(rl, bins=edges)[0]
                tot += max(t_lat(cal[F], int(n)) for n in per_rank)
            tot += (len(levels) * a.sync_us / 1e3) if N > 1 else 0.0
            out[N] = tot
            # ideal per-block readiness (no level barrier at all): the chain of
            # L dependent lone windows, or the busiest rank's throughput
            busiest = max(np.histogram(np.concatenate(row_of_level), bins=edges)[0])
            lb[N] = max(len(levels) * t_lat(cal[F], 1), t_lat(cal[F], int(busiest)))
        res[B] = {"F": F, "levels": len(levels), "blocks": plan.n_processed,
                  "model_ms": {n: round(v, 2) for n, v in out.items()},
                  "speedup": {n: round(out[1] / v, 2) for n, v in out.items()},
                  "dataflow_bound_ms": {n: round(v, 2) for n, v in lb.items()},
                  "dataflow_bound_speedup": {n: round(out[1] / v, 2) for n, v in lb.items()}}
        print(json.dumps({"B": B, **res[B]}), flush=True)
    return res


if __name__ == "__main__":
    main()
