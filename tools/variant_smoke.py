"""Small runs of every kernel variant in one process (a few windows, a few
iterations each), for use under a checker or after a kernel change.
(compute-sanitizer is closed on this GPU pool, so it has only been run plain.)
The cases cover the fast kernel at F = 32 / 64 / 128 in
fp32 and fp64 (narrow and wide level variants, lazy and tracked argmax), the
weight-spectrum cache (classification kernels, producer launch, cached twin
path), the reference-default kernel (DFT = window shape), the generic kernel
(odd DFT sizes, debug outputs), the dataflow executor, the strip shards, the
batched window entry point and the quantise/PSNR epilogue.

usage: python tools/variant_smoke.py [case ...]     (no argument: every case)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# the cache classifies every session, however small, in this process
os.environ.setdefault("FSE_WCACHE_ENTRIES", "1")
os.environ.setdefault("FSE_WCACHE_MIN_F", "32")
os.environ.setdefault("FSE_WCACHE_WIDTH", "0")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_00233_b200 as P  # noqa: E402
from paper_2207_00233_b200 import _lib, fse as fse_mod, synth  # noqa: E402
from paper_2207_00233_b200.conceal import conceal_batch, quantize_psnr_device  # noqa: E402

L = _lib.lib()
IT = int(os.environ.get("SAN_ITERS", "6"))


def scene(h, w, seed, kind="isolated", frac=0.3):
    img = synth.synthetic_frame(h, w, seed).astype(np.float64)
    m = synth.loss_mask(h, w, kind, frac, seed + 100)
    img[m == 1] = 0
    return img, m


def fast(prec, B, F, shape=(96, 130)):
    img, m = scene(*shape, seed=B + F)
    p = P.FseParams(d=min(14, (F - B) // 2), iterations=IT, block_size=B, fft_size=F)
    out, mo, rep = P.conceal(img, m, p, "optimized", precision=prec)
    assert np.isfinite(out).all() and rep.blocks_processed > 0
    return out


def wide(prec):
    """Levels wider than the SM count (the 6-warp throughput variants), through the batch path."""
    n = 6
    imgs, ms = zip(*[scene(128, 160, s, "mixed", 0.3) for s in range(n)])
    p = P.FseParams(d=14, iterations=IT, block_size=4, fft_size=64)
    out, mo, reps = conceal_batch(np.stack(imgs), np.stack(ms), p, precision=prec)
    assert np.isfinite(out).all()


CASES = {}


def case(f):
    CASES[f.__name__] = f
    return f


@case
def f32_b4_f64():
    fast("fp32", 4, 64)


@case
def f64_b4_f64():
    fast("fp64", 4, 64)


@case
def f32_b2_f32():
    fast("fp32", 2, 32, (64, 66))


@case
def f64_b2_f32():
    fast("fp64", 2, 32, (64, 66))


@case
def f32_b8_f128():
    fast("fp32", 8, 128)


@case
def f64_b8_f128():
    fast("fp64", 8, 128)


@case
def f32_wide_lazy():
    L.fse_set_track_below(0)  # lazy argmax on every level
    try:
        wide("fp32")
    finally:
        L.fse_set_track_below(16 * torch.cuda.get_device_properties(0).multi_processor_count)


@case
def f32_wide_tracked():
    wide("fp32")


@case
def f64_wide():
    wide("fp64")


@case
def f64_wide_nocache():
    L.fse_set_wcache(0)
    try:
        wide("fp64")
    finally:
        L.fse_set_wcache(1)


@case
def cache_every_map():
    os.environ["FSE_WCACHE_MIN"] = "1"
    os.environ["FSE_WCACHE_PLANES"] = "7"  # more maps than planes: the capacity path
    try:
        fast("fp64", 4, 64)
        fast("fp32", 4, 64)
    finally:
        os.environ.pop("FSE_WCACHE_MIN")
        os.environ.pop("FSE_WCACHE_PLANES")


@case
def defaults_gen():
    img, m = scene(130, 150, 5, "isolated", 0.3)
    p = P.FseParams(iterations=IT)  # d = 16, B = 16, DFT = window shape
    for prec in ("fp64", "fp32"):
        out, _, rep = P.conceal(img, m, p, precision=prec)
        assert np.isfinite(out).all() and rep.blocks_processed > 0


@case
def generic_odd():
    img, m = scene(90, 100, 6, "isolated", 0.3)
    p = P.FseParams(d=9, iterations=IT, block_size=5)  # 23 x 23 windows and clipped ones
    out, _, rep = P.conceal(img, m, p, "linescan", precision="fp64")
    assert np.isfinite(out).all() and rep.blocks_processed > 0


@case
def dataflow():
    L.fse_set_dataflow(1)
    try:
        fast("fp64", 4, 64)
        fast("fp32", 4, 64)
    finally:
        L.fse_set_dataflow(0)


@case
def windows_batch():
    rng = np.random.default_rng(3)
    v = rng.uniform(0, 255, (5, 30, 28))
    w = rng.uniform(0, 1, (5, 30, 28)) * (rng.uniform(size=(5, 30, 28)) > 0.3)
    for prec in ("fp64", "fp32"):
        fse_mod.run_fse_batch(v, w, IT, 0.5, precision=prec, fft_size=64)
    P.run_fse(v[0], w[0], IT, 0.5)


@case
def strips_one_rank():
    from paper_2207_00233_b200.strips import conceal_strips

    img, m = scene(160, 128, 9, "burst2d", 0.4)
    p = P.FseParams(d=14, iterations=IT, block_size=4, fft_size=64)
    out = conceal_strips(img, m, p, precision="fp64")
    assert np.isfinite(out[0]).all()


@case
def epilogue():
    img, m = scene(64, 96, 11)
    x = torch.from_numpy(np.stack([img, img])).cuda()
    t = torch.from_numpy(np.clip(np.stack([img, img]) + 1.0, 0, 255).astype(np.uint8)).cuda()
    mk = torch.from_numpy(np.stack([m, m])).cuda()
    quantize_psnr_device(x, t, mk)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        torch.cuda.synchronize()
        print("ok", n, flush=True)
