"""For fuzz_parity seeds whose result differs from the oracle: find the first
block (in the oracle's processing order) whose canonical pick sequence differs,
re-run that block's greedy selection in numpy float64 on the oracle's inputs and
print, at the first differing iteration, the energies of the two candidates --
the oracle's pick and the device's -- and their relative margin.  A margin at
rounding level (<~1e-13) is a tie that the DFT's rounding decides (the reference
computes fft2, the device a separable DFT); a large margin is a device bug.

usage: python tests/fuzz_debug.py seed [seed ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2207_00233_b200 as P  # noqa: E402
from fuzz_parity import fft_shape, make_case  # noqa: E402
from oracle import oracle as O  # noqa: E402


def greedy(vpad, wpad, iterations, gamma, forced=None):
    """_kernel.pyx:128-187 in numpy (fft2 set-up, first maximum in row-major
    order, the two-term update).  forced: a pick list to follow instead of the
    argmax (to evaluate another sequence's candidates); returns per-iteration
    (pick, energy plane)."""
    F1, F2 = vpad.shape
    W = np.fft.fft2(wpad)
    R = np.fft.fft2(np.where(wpad > 0, vpad, 0.0) * wpad)
    tot = W[0, 0].real
    out = []
    for it in range(iterations):
        e = R.real ** 2 + R.imag ** 2
        k = int(np.argmax(e))  # first maximum, row-major (strict '>')
        a, b = divmod(k, F2)
        out.append(((a, b), e.copy()))
        if forced is not None:
            a, b = forced[it]
        p = R[a, b] / tot
        ia = (np.arange(F1)[:, None] - a) % F1
        ib = (np.arange(F2)[None, :] - b) % F2
        ja = (np.arange(F1)[:, None] + a) % F1
        jb = (np.arange(F2)[None, :] + b) % F2
        selfc = (2 * a) % F1 == 0 and (2 * b) % F2 == 0
        if selfc:
            R = R - gamma * p.real * W[ia, ib]
        else:
            R = R - gamma * (p * W[ia, ib] + np.conj(p) * W[ja, jb])
    return out


def debug(seed):
    kind, img, mask, par, fft, order = make_case(seed)
    fs = fft_shape(fft, par["block_size"], par["d"])
    p = P.FseParams(fft_size=fft, **par)
    out, om, rep, picks = P.conceal(img, mask, p, order, precision="fp64", return_picks=True)
    op = O.Params(fft_size=fs, **par)
    calls = []
    real_extrapolate = O.extrapolate

    def spy(values, cls, rect, pp, kernel="auto", want_picks=False):
        res = real_extrapolate(values, cls, rect, pp, kernel, want_picks)
        calls.append((np.array(values, copy=True), np.array(cls, copy=True), rect, res))
        return res

    O.extrapolate = spy
    try:
        ref, rm, rrep = O.conceal(img, mask, op, order, want_picks=True, kernel="auto")
    finally:
        O.extrapolate = real_extrapolate
    err = float(np.max(np.abs(out - ref)))
    print(f"seed {seed}: {kind} {img.shape} B={par['block_size']} d={par['d']} fft={fft} I={par['iterations']} "
          f"rho={par['rho']} delta={par['delta']} gamma={par['gamma']} {order}: max sample error {err:.3g}")
    fitted = [c for c in calls if (c[3][0] if isinstance(c[3], tuple) else c[3]) is not None]
    # compare per block in dictionary order of the oracle's picks (insertion = processing order)
    for idx, (b, pk) in enumerate(rrep.picks.items()):
        m, n = fitted[idx][0].shape
        shape = fs if fs is not None else (m, n)
        dev = O.canonical_picks(picks[b], shape)
        want = O.canonical_picks(pk, shape)
        if dev == want:
            continue
        it = next(i for i, (x, y) in enumerate(zip(dev, want)) if x != y)
        values, cls, rect, _ = fitted[idx]
        w = O.weight_plane(values.shape, cls, par["rho"], par["delta"])
        vpad = np.zeros(shape)
        wpad = np.zeros(shape)
        vpad[:m, :n] = values
        wpad[:m, :n] = w
        hist = greedy(vpad, wpad, it + 1, par["gamma"], forced=[tuple(x) for x in want[:it]] + [tuple(want[it])])
        e = hist[it][1]
        ew, ed = e[tuple(want[it])], e[tuple(dev[it])]
        known = int((w > 0).sum())
        margin = (ew - ed) / max(ew, 1e-300)
        e0 = float(hist[0][1].max())
        print(f"   first differing block {b} (#{idx} in order), window {values.shape} with {known} weighted samples, "
              f"iteration {it}: oracle pick {tuple(want[it])} energy {ew:.17g}, device pick {tuple(dev[it])} "
              f"energy {ed:.17g}, relative margin {margin:.3g}, energy / initial maximum {ew / max(e0, 1e-300):.3g}; "
              f"numpy argmax {hist[it][0]}")
        # a tie: the candidates agree to rounding level, or the residual has already
        # converged to rounding noise (energy below 1e-16 of its start, i.e. amplitudes
        # below 1e-8 of it: what is left is the DFT's own rounding, which differs
        # between fft2 and the device's separable DFT)
        return {"margin": margin, "noise": ew / max(e0, 1e-300), "err": err,
                "tie": abs(margin) < 1e-9 or ew <= 1e-16 * max(e0, 1e-300)}
    print("   picks identical for every block (difference is not a pick switch)")
    return {"margin": None, "noise": None, "err": err, "tie": False}


if __name__ == "__main__":
    for s in sys.argv[1:]:
        try:
            debug(int(s))
        except Exception as e:  # noqa: BLE001
            print(f"seed {s}: debug failed: {type(e).__name__}: {e}")
