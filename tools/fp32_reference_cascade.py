"""Is the north_star's fp32 contract reachable by ANY fp32 implementation?

Test infrastructure / evidence (CPU only, imports oracle/): the reference's own
algorithm, computed in float32 -- numpy restatement of run_fse/_iterate
(/root/reference/pkg/src/fsefill/_kernel.pyx:14-187) with every spectrum,
weight spectrum, coefficient and energy in float32, the setup fft2 in
single precision (numpy >= 2 keeps complex64), the strict-'>' first-maximum
scan and the same update order -- driven through the oracle's restatement of
conceal() (oracle/oracle.py, conceal.py:97-181), i.e. exactly the reference
pipeline with its kernel in fp32.  It is compared with the fp64 reference
(oracle/_ref, the reference's compiled kernel) on the same inputs.

If this "fp32 reference" also misses "every lost sample within 0.5, PSNR
within 0.02 dB", the miss is a property of the greedy selection in fp32, not
of the B200 kernels: a switched pick in one block feeds every later block
that reads it as R.

usage: python tools/fp32_reference_cascade.py [--config 1|2] [--order optimized|linescan]
       [--blocks N] [--json out.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import oracle as O  # noqa: E402
from paper_2207_00233_b200 import synth  # noqa: E402


def run_fse_f32(values, weights, iterations, gamma):
    """_kernel.pyx:128-187 + _iterate in float32 (vectorised over the spectrum).

    Returns (coeff complex128, picks, energies, residual) like run_fse, the
    coefficients accumulated in float32 and widened at the end."""
    f = np.float32
    v = np.asarray(values, np.float32)
    w = np.asarray(weights, np.float32)
    m, n = v.shape
    tot = f(np.sum(w, dtype=np.float32))
    r = np.where(w > 0, v, f(0)).astype(np.float32)
    g = np.fft.fft2(w * r).astype(np.complex64)  # _kernel.pyx:147
    W = np.fft.fft2(w).astype(np.complex64)  # _kernel.pyx:148
    g_re = g.real.copy()
    g_im = g.imag.copy()
    wf_re = W.real
    wf_im = W.imag
    c_re = np.zeros((m, n), np.float32)
    c_im = np.zeros((m, n), np.float32)
    gam = f(gamma)
    picks = np.zeros((iterations, 2), np.int32)
    uu = np.arange(m)[:, None]
    vv = np.arange(n)[None, :]
    for it in range(iterations):
        e = g_re * g_re + g_im * g_im  # float32, first maximum in row-major order
        k = int(np.argmax(e))  # np.argmax returns the first occurrence (strict '>')
        a, b = divmod(k, n)
        picks[it] = (a, b)
        p_re = g_re[a, b] / tot
        p_im = g_im[a, b] / tot
        lo_r = wf_re[(uu - a) % m, (vv - b) % n]
        lo_i = wf_im[(uu - a) % m, (vv - b) % n]
        if (2 * a) % m == 0 and (2 * b) % n == 0:
            c_re[a, b] += gam * p_re
            g_re -= gam * p_re * lo_r
            g_im -= gam * p_re * lo_i
        else:
            c_re[a, b] += gam * p_re
            c_im[a, b] += gam * p_im
            iu, iv = (m - a) % m, (n - b) % n
            c_re[iu, iv] += gam * p_re
            c_im[iu, iv] -= gam * p_im
            hi_r = wf_re[(uu + a) % m, (vv + b) % n]
            hi_i = wf_im[(uu + a) % m, (vv + b) % n]
            t_re = p_re * (lo_r + hi_r) - p_im * (lo_i - hi_i)
            t_im = p_re * (lo_i + hi_i) + p_im * (lo_r - hi_r)
            g_re -= gam * t_re
            g_im -= gam * t_im
    coeff = c_re.astype(np.float64) + 1j * c_im.astype(np.float64)
    return coeff, picks, np.zeros(iterations + 1), np.zeros((m, n))


def psnr(ref, img, mask):
    region = mask != 0  # the concealed samples, as evalkit.psnr (evalkit.py:67-81)
    err = np.mean((ref[region] - img[region]) ** 2)
    return 10 * np.log10(255.0 ** 2 / err) if err > 0 else float("inf")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--order", default="optimized")
    ap.add_argument("--blocks", type=int, default=0, help="stop after this many fitted blocks (0 = all)")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    img, mask = synth.config_scene(a.config)
    orig = img.copy()
    p = O.Params(d=14, rho=0.8, delta=0.2, gamma=0.5, iterations=100, block_size=4, fft_size=(64, 64))
    lim = a.blocks or None

    t0 = time.perf_counter()
    ref, rmask, rrep = O.conceal(img, mask, p, a.order, kernel="ref", want_picks=True, block_limit=lim)
    t1 = time.perf_counter()
    saved = O.run_fse
    O.run_fse = lambda v, w, i, g, kernel="auto": run_fse_f32(v, w, i, g)
    try:
        f32, fmask, frep = O.conceal(img, mask, p, a.order, kernel="ref", want_picks=True, block_limit=lim)
    finally:
        O.run_fse = saved
    t2 = time.perf_counter()

    lost = mask == O.LOST
    d = np.abs(f32 - ref)[lost]
    switched = [b for b, pk in rrep.picks.items()
                if O.canonical_picks(pk, (64, 64)) != O.canonical_picks(frep.picks.get(b, []), (64, 64))]
    # first block (in processing order) whose picks differ, and how many
    # earlier-processed blocks it had as R inputs: the cascade's seed
    order = [b for batch in rrep.batches for b in batch]
    first = next((b for b in order if b in set(switched)), None)
    res = {
        "what": "reference algorithm in float32 (numpy restatement of _kernel.pyx) vs the fp64 reference kernel (oracle/_ref), same conceal() pipeline",
        "config": a.config,
        "order": a.order,
        "blocks": len(rrep.picks),
        "blocks_with_switched_picks": len(switched),
        "first_switched_block_in_processing_order": first,
        "first_switch_position": order.index(first) if first is not None else None,
        "lost_samples": int(lost.sum()),
        "max_abs": float(d.max()) if d.size else 0.0,
        "share_above_0.5": float(np.mean(d > 0.5)) if d.size else 0.0,
        "psnr_fp64_db": psnr(orig.astype(np.float64), ref, mask),
        "psnr_fp32_db": psnr(orig.astype(np.float64), f32, mask),
        "seconds": {"fp64": round(t1 - t0, 1), "fp32": round(t2 - t1, 1)},
    }
    res["delta_psnr_db"] = res["psnr_fp32_db"] - res["psnr_fp64_db"]
    print(json.dumps(res))
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
