"""Dev (CPU): how often reduced-precision variants of the FSE recurrence switch a
pick relative to the fp64 reference kernel -- the question behind the fp32
tolerance.

Windows: the first-batch windows of BASELINE config 1 / config 3 (isolated
losses, classes from the original mask), zero-padded to F = 64, I = 100.
Reference: oracle/_ref (the reference's own compiled _kernel.pyx).
Variants, numpy emulations of the incremental update (_kernel.pyx:31-97):
  f64      : fp64 throughout (sanity: should agree up to near-ties at 1e-15)
  mixed    : g accumulated in fp64, W (and the initial spectra) rounded to fp32
             (the variant VERDICT r1 asked for)
  f32      : g, W, p and the update in fp32
Reports, per variant, the share of windows whose canonical pick sequence
differs from the reference and the distribution of the first divergence.
usage: python tools/fp32_pick_study.py [n_windows] [config]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import oracle as O
from paper_2207_00233_b200 import synth


def emulate(values, weights, iters, gamma, g_dt, w_dt):
    F1, F2 = values.shape
    x = np.where(weights > 0, values, 0.0) * weights
    g = np.fft.fft2(x).astype(np.complex128).astype(g_dt)
    W = np.fft.fft2(weights).astype(w_dt)
    tot = weights.sum()
    picks = []
    uu = np.arange(F1)[:, None]
    vv = np.arange(F2)[None, :]
    for _ in range(iters):
        e = (g.real.astype(np.float64) ** 2 + g.imag.astype(np.float64) ** 2) if g_dt == np.complex128 else (
            g.real * g.real + g.imag * g.imag)
        k = int(np.argmax(e))
        a, b = divmod(k, F2)
        picks.append((a, b))
        p = g[a, b] / g_dt(tot) if g_dt == np.complex64 else g[a, b] / tot
        selfc = (2 * a) % F1 == 0 and (2 * b) % F2 == 0
        Wm = W[(uu - a) % F1, (vv - b) % F2]
        if selfc:
            g = g - (gamma * p.real) * Wm.astype(g.dtype)
        else:
            Wp = W[(uu + a) % F1, (vv + b) % F2]
            g = g - gamma * (p * Wm.astype(g.dtype) + np.conj(p) * Wp.astype(g.dtype))
        g = g.astype(g_dt)
    return picks


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    img, mask = synth.config_scene(cfg)
    img = img.astype(np.float64)
    p = O.Params(d=14, rho=0.8, delta=0.2, gamma=0.5, iterations=100, block_size=4, fft_size=(64, 64))
    grid = O.Grid.of(mask.shape[0], mask.shape[1], 4)
    lossy = np.flatnonzero(O.lost_per_block(grid, mask).reshape(-1) > 0)
    rng = np.random.default_rng(0)
    sel = rng.choice(lossy, size=min(n, lossy.size), replace=False)
    res = {k: [] for k in ("f64", "mixed", "f32")}
    for b in sel:
        origin, cls, rect = O.classify(grid, mask, int(b), p.d)
        m, nn = cls.shape
        vals = img[origin[0]:origin[0] + m, origin[1]:origin[1] + nn]
        w = O.weight_plane((m, nn), cls, p.rho, p.delta)
        vp = np.zeros((64, 64)); wp = np.zeros((64, 64))
        vp[:m, :nn] = vals
        wp[:m, :nn] = w
        if not (wp > 0).any():
            continue
        _, ref_picks, _, _ = O.run_fse(vp, wp, 100, 0.5)
        ref = O.canonical_picks(ref_picks, (64, 64))
        for name, gdt, wdt in (("f64", np.complex128, np.complex128), ("mixed", np.complex128, np.complex64),
                               ("f32", np.complex64, np.complex64)):
            pk = O.canonical_picks(emulate(vp, wp, 100, 0.5, gdt, wdt), (64, 64))
            first = next((i for i, (x, y) in enumerate(zip(pk, ref)) if x != y), None)
            res[name].append(first)
    for name, v in res.items():
        bad = [f for f in v if f is not None]
        print(f"{name:6s}: {len(bad)}/{len(v)} windows switch a pick ({100 * len(bad) / max(1, len(v)):.1f}%)"
              + (f", first switch at iteration median {int(np.median(bad))}, min {min(bad)}" if bad else ""))


if __name__ == "__main__":
    main()
