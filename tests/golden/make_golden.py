"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref built by
oracle/build_ref.sh):   python tests/golden/make_golden.py

The reference package (/root/reference/pkg/src/fsefill) is imported as-is; its
compiled backend is the reference's own _kernel.pyx compiled into oracle/_ref.
For FFT sizes larger than the window the reference's extrapolate_block is
wrapped by the top-left zero-padding adapter of SURVEY.md §8(c) (patched on
sys.modules["fsefill.conceal"], since fsefill.conceal is the function,
fsefill/__init__.py:4).  Nothing here is used at run time; only the .npz files
it writes are committed.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import fsefill  # noqa: E402
from fsefill import fse  # noqa: E402
from fsefill.fse import FseParams, weight_plane  # noqa: E402
from fsefill.grid import AREA_A, AREA_BI, AREA_BO, AREA_R  # noqa: E402
from fsefill.schedule import init_counts, schedule_all  # noqa: E402
from fsefill.grid import build_grid  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2207_00233_b200 import synth  # noqa: E402

fse._BACKENDS["compiled"] = O.ref_kernel()
fse.set_backend("compiled")
conceal_mod = sys.modules["fsefill.conceal"]
_native_extrapolate = conceal_mod.extrapolate_block
RECORD: dict = {}


def make_adapter(F, grid_B, cols):
    def extrapolate_padded(win, params):
        values = np.ascontiguousarray(win.values, dtype=np.float64)
        w = weight_plane(values.shape, win.cls, params)
        if not (w > 0.0).any():
            raise fse.DegenerateWindowError("window has no usable samples")
        m, n = values.shape
        F1, F2 = (m, n) if F is None else F
        vp = np.zeros((F1, F2)); wp = np.zeros((F1, F2))
        vp[:m, :n] = values
        wp[:m, :n] = w
        coeff, picks, _, _ = fse._BACKENDS["compiled"].run_fse(vp, wp, params.iterations, params.gamma)
        syn = (np.fft.ifft2(coeff) * (F1 * F2)).real[:m, :n]
        r0, r1, c0, c1 = win.block_rect
        b = ((win.origin[0] + r0) // grid_B) * cols + (win.origin[1] + c0) // grid_B
        RECORD[b] = np.asarray(O.canonical_picks(picks, (F1, F2)), dtype=np.int32)
        return syn[r0:r1, c0:c1].copy()
    return extrapolate_padded


def run_fse_cases():
    out = {}
    k = fse._BACKENDS["compiled"]
    cases = []
    # (a) the reference's own kernel-test shapes (test_fse.py:106-129 style)
    for seed in range(6):
        rng = np.random.default_rng(100 + seed)
        m, n = int(rng.integers(4, 20)), int(rng.integers(4, 20))
        v = rng.uniform(0.0, 255.0, (m, n))
        w = rng.uniform(0.0, 1.0, (m, n))
        w[rng.uniform(size=(m, n)) < 0.35] = 0.0
        w[m // 2, n // 2] = 1.0
        cases.append((v, w, 25, 0.5))
    # (b) FSE windows from a synthetic scene, zero-padded to F x F (B=2/4/8, d=14)
    img, mask = synth.config_scene(1)
    img = img.astype(np.float64)
    rng = np.random.default_rng(7)
    for F, msz, iters in ((32, 30, 60), (64, 32, 100), (64, 22, 100), (128, 36, 40)):
        r, c = int(rng.integers(0, 400)), int(rng.integers(0, 400))
        v = img[r : r + msz, c : c + msz].copy()
        cls = np.full((msz, msz), AREA_A, dtype=np.uint8)
        lo = (msz - 4) // 2
        cls[lo : lo + 4, lo : lo + 4] = AREA_BI
        cls[rng.uniform(size=(msz, msz)) < 0.1] = AREA_R
        cls[rng.uniform(size=(msz, msz)) < 0.05] = AREA_BO
        w = weight_plane((msz, msz), cls, FseParams(rho=0.8, delta=0.2))
        vp = np.zeros((F, F)); wp = np.zeros((F, F))
        vp[:msz, :msz] = v
        wp[:msz, :msz] = w
        cases.append((vp, wp, iters, 0.5))
    for i, (v, w, it, g) in enumerate(cases):
        coeff, picks, en, res = k.run_fse(v, w, it, g)
        out[f"c{i}_values"] = v
        out[f"c{i}_weights"] = w
        out[f"c{i}_meta"] = np.array([it, g])
        out[f"c{i}_coeff"] = coeff
        out[f"c{i}_picks"] = picks
        out[f"c{i}_canon"] = np.asarray(O.canonical_picks(picks, v.shape), dtype=np.int32)
        out[f"c{i}_energies"] = en
        out[f"c{i}_residual"] = res
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "run_fse_cases.npz"), **out)


def schedule_cases():
    out = {}
    rng = np.random.default_rng(0)
    n = 0
    shapes = [(3, 3, 1.0), (1, 1, 1.0), (2, 2, 0.0)] + [
        (int(rng.integers(1, 17)), int(rng.integers(1, 17)), float(rng.uniform(0.05, 1.0)))
        for _ in range(40)
    ] + [(68, 120, 0.2), (128, 128, 0.3)]
    for rows, cols, dens in shapes:
        table = (rng.uniform(size=(rows, cols)) < dens).astype(np.int64)
        if (rows, cols) == (3, 3):
            table[:] = 1
        g = build_grid(cols * 4, rows * 4, 4)
        counts = init_counts(g, table)
        batches = schedule_all(g, counts)
        out[f"s{n}_table"] = table.astype(np.uint8)
        out[f"s{n}_counts"] = counts
        out[f"s{n}_ptr"] = np.cumsum([0] + [len(b) for b in batches]).astype(np.int32)
        out[f"s{n}_blocks"] = np.asarray([b for bt in batches for b in bt], dtype=np.int32)
        n += 1
    out["n_cases"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "schedule_cases.npz"), **out)


def scene(h, w):
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)
    return 120.0 + 50.0 * np.sin(x / 5.0) + 30.0 * np.cos(y / 7.0) + 0.3 * x


def conceal_cases():
    from fsefill.conceal import conceal
    out = {}
    cases = []
    # (name, image, mask, params, order, F)
    m1 = np.zeros((64, 64), np.uint8)
    m1[10:24, 10:24] = 1; m1[28:44, 36:52] = 1; m1[44:52, 4:12] = 1
    for order in ("optimized", "linescan"):
        cases.append((f"native_{order}", scene(64, 64), m1, FseParams(d=8, iterations=30, block_size=8), order, None))
    img, mask = synth.config_scene(1)
    img = img[:128, :160].astype(np.float64).copy()
    mask = mask[:128, :160].copy()
    mask[:] = 0
    rng = np.random.default_rng(5)
    for _ in range(10):
        r, c = int(rng.integers(1, 7)) * 16, int(rng.integers(1, 9)) * 16
        mask[r : r + 16, c : c + 16] = 1
    for order in ("optimized", "linescan"):
        cases.append((f"f64_{order}", img, mask, FseParams(d=14, iterations=100, block_size=4), order, (64, 64)))
    img2, mask2 = synth.config_scene(2)
    img2 = img2[:96, :128].astype(np.float64).copy(); mask2 = mask2[:96, :128].copy()
    for order in ("optimized", "linescan"):
        cases.append((f"burst_{order}", img2, mask2, FseParams(d=14, iterations=60, block_size=4), order, (64, 64)))
    cases.append(("b2_f32", img[:64, :64].copy(), mask[:64, :64].copy(), FseParams(d=14, iterations=50, block_size=2), "optimized", (32, 32)))
    cases.append(("b8_f128", img[:96, :96].copy(), mask[:96, :96].copy(), FseParams(d=14, iterations=30, block_size=8), "optimized", (128, 128)))
    # ragged image edges, partial blocks, native clipped windows
    m3 = np.zeros((37, 53), np.uint8)
    m3[3:9, 40:53] = 1; m3[20:37, 0:7] = 1; m3[14:16, 22:30] = 1
    cases.append(("ragged_native", scene(37, 53), m3, FseParams(d=6, iterations=20, block_size=8), "optimized", None))
    # hole peeled by retry sweeps (test_conceal.py:187-199)
    m4 = np.zeros((96, 96), np.uint8); m4[16:80, 16:80] = 1
    cases.append(("hole_retry", scene(96, 96), m4, FseParams(d=4, iterations=20, block_size=8), "optimized", None))
    # all lost (test_conceal.py:177-184)
    cases.append(("all_lost", scene(32, 32), np.ones((32, 32), np.uint8), FseParams(d=8, iterations=30, block_size=8), "optimized", None))
    for i, (name, im, mk, p, order, F) in enumerate(cases):
        g = build_grid(im.shape[1], im.shape[0], p.block_size)
        conceal_mod.extrapolate_block = make_adapter(F, p.block_size, g.cols)
        RECORD.clear()
        o_img, o_mask, rep = conceal(im, mk, p, order)
        out[f"k{i}_name"] = np.array(name)
        out[f"k{i}_image"] = im
        out[f"k{i}_mask"] = mk
        out[f"k{i}_params"] = np.array([p.d, p.rho, p.delta, p.gamma, p.iterations, p.block_size])
        out[f"k{i}_order"] = np.array(order)
        out[f"k{i}_fft"] = np.array(F if F is not None else (0, 0))
        out[f"k{i}_out_image"] = o_img
        out[f"k{i}_out_mask"] = o_mask
        out[f"k{i}_batch_ptr"] = np.cumsum([0] + [len(b) for b in rep.batches]).astype(np.int32)
        out[f"k{i}_batch_blocks"] = np.asarray([b for bt in rep.batches for b in bt], dtype=np.int32)
        out[f"k{i}_unconcealed"] = np.asarray(rep.unconcealed_blocks, dtype=np.int32)
        out[f"k{i}_processed"] = np.array(rep.blocks_processed)
        keys = sorted(RECORD)
        out[f"k{i}_pick_blocks"] = np.asarray(keys, dtype=np.int32)
        out[f"k{i}_picks"] = (np.stack([RECORD[b] for b in keys]) if keys else np.zeros((0, p.iterations, 2), np.int32))
        conceal_mod.extrapolate_block = _native_extrapolate
        print(name, order, rep.blocks_processed, len(rep.batches), rep.unconcealed_blocks[:5])
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "conceal_cases.npz"), **out)


def weight_cases():
    p = FseParams()
    out = {}
    rng = np.random.default_rng(11)
    for i, (m, n) in enumerate(((9, 14), (9, 9), (4, 6), (18, 32), (32, 32), (36, 22))):
        cls = rng.choice(np.array([AREA_A, AREA_BI, AREA_BO, AREA_R], dtype=np.uint8), size=(m, n))
        out[f"w{i}_cls"] = cls
        out[f"w{i}_plane"] = weight_plane((m, n), cls, p)
    out["n_cases"] = np.array(6)
    np.savez_compressed(os.path.join(HERE, "weight_cases.npz"), **out)


def full_config_cases():
    """BASELINE configs 1 and 2 at full size (512 x 512, F=64, I=100, d=14, B=4)
    through the reference pipeline; only the lost samples, the batches and the
    per-block canonical picks are stored (the inputs are regenerated from the
    seeded generator in paper_2207_00233_b200/synth.py)."""
    from fsefill.conceal import conceal
    out = {}
    cases = [("cfg1_optimized", 1, "optimized"), ("cfg2_optimized", 2, "optimized"),
             ("cfg2_linescan", 2, "linescan")]
    p = FseParams(d=14, iterations=100, block_size=4)
    for i, (name, cfg, order) in enumerate(cases):
        img, mask = synth.config_scene(cfg)
        g = build_grid(img.shape[1], img.shape[0], 4)
        conceal_mod.extrapolate_block = make_adapter((64, 64), 4, g.cols)
        RECORD.clear()
        o_img, o_mask, rep = conceal(img.astype(np.float64), mask, p, order)
        lost = mask == 1
        out[f"f{i}_name"] = np.array(name)
        out[f"f{i}_config"] = np.array(cfg)
        out[f"f{i}_order"] = np.array(order)
        out[f"f{i}_image_sum"] = np.array([int(img.astype(np.int64).sum()), int(mask.astype(np.int64).sum())])
        out[f"f{i}_lost_values"] = o_img[lost]
        out[f"f{i}_out_mask_sum"] = np.array(int(o_mask.astype(np.int64).sum()))
        out[f"f{i}_batch_ptr"] = np.cumsum([0] + [len(b) for b in rep.batches]).astype(np.int32)
        out[f"f{i}_batch_blocks"] = np.asarray([b for bt in rep.batches for b in bt], dtype=np.int32)
        keys = sorted(RECORD)
        out[f"f{i}_pick_blocks"] = np.asarray(keys, dtype=np.int32)
        out[f"f{i}_picks"] = np.stack([RECORD[b] for b in keys]).astype(np.uint8)
        conceal_mod.extrapolate_block = _native_extrapolate
        print(name, rep.blocks_processed, len(rep.batches))
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "full_cfg.npz"), **out)


if __name__ == "__main__":
    run_fse_cases()
    schedule_cases()
    weight_cases()
    conceal_cases()
    full_config_cases()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
