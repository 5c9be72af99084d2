"""Scaling model of config-5 strip sharding, from measured inputs.

usage: python tools/scaling_model.py LATENCY.jsonl [--precision fp32|fp64] [--sync-us 4]

Inputs:
  * LATENCY.jsonl: tools/window_latency.py on a B200 -- the device time of one
    dependency level holding n independent windows, per FFT size/precision;
  * the real config-5 plan (C++ planner, run here): every block's dependency
    level, and the row bands strips.band_partition gives N ranks.
Model (per-level halo protocol, round 1): a rank runs level l after its
neighbours finished level l-1, so the step is
    T(N) = sum_l max_r T_lat(n_{l,r}) + L * t_sync(N)
with n_{l,r} the rank's windows of level l and T_lat interpolated from the
measured level times (piecewise linear in n, waves beyond the largest
measured n).  Dependency-exact protocol (round 2, the one built): a rank
starts level l after its own level l-1 and after each neighbour has finished
the levels its level-l windows read (halo_needs), simulated rank by rank.  t_sync(1) = 0.  The same sum at N = 1 is checked against the
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


def halo_needs(lev, rank, lo, hi, R):
    """Per level of band [lo, hi): the neighbour levels (+1) its windows read
    (fse_cuda.cu session_open: need_up / need_down), 0 = none."""
    rows, cols = lev.shape
    L = int(lev.max()) + 1
    out = []
    for z0, z1, n0, n1 in ((lo, min(hi, lo + R), max(0, lo - R), lo), (max(lo, hi - R), hi, hi, min(rows, hi + R))):
        need = np.zeros(L, np.int64)
        if n1 <= n0 or z1 <= z0:
            out.append(need)
            continue
        lb, rb = lev[z0:z1], rank[z0:z1]
        nb = np.zeros_like(lb)
        for dr in range(-R, R + 1):
            for dc in range(-R, R + 1):
                rr = np.arange(z0, z1) + dr
                ok_r = (rr >= n0) & (rr < n1)
                if not ok_r.any():
                    continue
                cc = np.arange(cols) + dc
                ok_c = (cc >= 0) & (cc < cols)
                lo_ = lev[np.clip(rr, 0, rows - 1)][:, np.clip(cc, 0, cols - 1)]
                ro_ = rank[np.clip(rr, 0, rows - 1)][:, np.clip(cc, 0, cols - 1)]
                m = ok_r[:, None] & ok_c[None, :] & (lo_ >= 0) & (ro_ < rb) & (lb >= 0)
                nb = np.maximum(nb, np.where(m, lo_ + 1, 0))
        sel = lb >= 0
        np.maximum.at(need, lb[sel], nb[sel])
        out.append(need)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("latency")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--sync-us", type=float, default=4.0,
                    help="per-level neighbour flag wait at N > 1 (cuStreamWaitValue32 + signal kernel)")
    ap.add_argument("--balance", action="store_true",
                    help="balance the plan's levels for N GPUs (fse_plan_rebalance with N x the one-GPU capacities)")
    ap.add_argument("--sms", type=int, default=148)
    a = ap.parse_args()
    cal = load(a.latency, a.precision)
    img, mask = synth.config_scene(5)
    res = {}
    for B, F in ((2, 32), (4, 64), (8, 128)):
        if F not in cal:
            continue
        p = P.FseParams(d=14, iterations=100, block_size=B, fft_size=F)
        R = strips.halo_rows(p)
        out, lb, ex = {}, {}, {}
        per_sm = {("fp64", 64): 3, ("fp32", 64): 4, ("fp64", 32): 6, ("fp32", 32): 8}.get((a.precision, F), 1)
        for N in (1, 2, 4, 8):
            plan = P.build_plan(mask, p)
            if a.balance:
                plan.rebalance(a.sms * N, a.sms * per_sm * N)
            rows, cols = plan.rows, plan.cols
            levels = plan.levels()
            processed = (plan.ranks() != np.iinfo(np.int32).max).reshape(rows, cols)
            row_of_level = [np.asarray(lv, np.int64) // cols for lv in levels]
            lev = np.full(rows * cols, -1, np.int64)
            for l, blk in enumerate(levels):
                lev[np.asarray(blk, np.int64)] = l
            lev = lev.reshape(rows, cols)
            rank = plan.ranks().astype(np.int64).reshape(rows, cols)
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
            # dependency-exact waits (the protocol built): rank r starts level l
            # after its own level l-1 and after each neighbour finished the
            # levels its level-l windows read (need_up / need_down)
            L = len(levels)
            per = np.array([np.histogram(rl, bins=edges)[0] for rl in row_of_level])  # [L, N]
            needs = [halo_needs(lev, rank, bands[r][0], bands[r][1], R) for r in range(N)]
            end = np.zeros((N, L))
            for l in range(L):
                for r in range(N):
                    t0 = end[r, l - 1] if l else 0.0
                    up, down = needs[r]
                    if r > 0 and up[l] > 0:
                        t0 = max(t0, end[r - 1, up[l] - 1] + a.sync_us / 1e3)
                    if r + 1 < N and down[l] > 0:
                        t0 = max(t0, end[r + 1, down[l] - 1] + a.sync_us / 1e3)
                    end[r, l] = t0 + t_lat(cal[F], int(per[l, r]))
            ex[N] = float(end[:, -1].max())
        res[B] = {"F": F, "levels": len(levels), "blocks": plan.n_processed,
                  "model_ms": {n: round(v, 2) for n, v in out.items()},
                  "speedup": {n: round(out[1] / v, 2) for n, v in out.items()},
                  "dependency_exact_ms": {n: round(v, 2) for n, v in ex.items()},
                  "dependency_exact_speedup": {n: round(out[1] / v, 2) for n, v in ex.items()},
                  "dataflow_bound_ms": {n: round(v, 2) for n, v in lb.items()},
                  "dataflow_bound_speedup": {n: round(out[1] / v, 2) for n, v in lb.items()}}
        print(json.dumps({"B": B, **res[B]}), flush=True)
    return res


if __name__ == "__main__":
    main()
