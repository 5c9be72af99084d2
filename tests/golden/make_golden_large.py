"""Full-size golden outputs from the REFERENCE itself (round 2 additions).

Run in the build container (needs /root/reference and oracle/_ref built by
oracle/build_ref.sh):   python tests/golden/make_golden_large.py [case ...]

Same method as make_golden.py: the unmodified reference package
(/root/reference/pkg/src/fsefill) with its compiled kernel, the F-adapter of
SURVEY.md §8(c) patched on sys.modules["fsefill.conceal"] for F > window.
Each case runs in its own process (the reference pipeline is sequential).

Cases (inputs are regenerated from the seeded generators in
paper_2207_00233_b200/synth.py; only outputs are stored):
  cfg3        BASELINE config 3: 1920x1080, 30% isolated, B=4 d=14 F=64 I=200
  cfg4f0      BASELINE config 4, frame 0: 1920x1080, 20% mixed, B=4 d=14 F=64 I=100
  cfg5crop    BASELINE config 5 (4K, 50% 2-D bursts) crop rows 0:768, cols 0:1024,
              B=4 d=14 F=64 I=100
  cfg3def     config 3's frame and mask with the reference's DEFAULT parameters
              (FseParams(): B=16 d=16 I=200, DFT = window size) -- the drop-in
              call conceal(image, mask) with no params
Stored per case: lost-sample values (float64, row-major over mask == LOST),
the batches (CSR), the output-mask checksum, and per block a 64-bit FNV-1a
hash of its canonical pick sequence (tests/reference.py:59-71 folding) plus
the full canonical picks of every 16th block.
"""

from __future__ import annotations

import os
import sys
from multiprocessing import get_context

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

CASES = {
    # name: (config, frame, crop, params kwargs, fft)
    "cfg3": (3, 0, None, dict(d=14, iterations=200, block_size=4), (64, 64)),
    "cfg4f0": (4, 0, None, dict(d=14, iterations=100, block_size=4), (64, 64)),
    "cfg5crop": (5, 0, (0, 768, 0, 1024), dict(d=14, iterations=100, block_size=4), (64, 64)),
    "cfg3def": (3, 0, None, dict(), None),
}


def pick_hash(canon) -> int:
    """64-bit FNV-1a over the (a, b) pairs of a canonical pick sequence."""
    h = 0xCBF29CE484222325
    for a, b in canon:
        for v in (int(a), int(b)):
            h ^= v & 0xFFFF
            h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h - (1 << 64) if h >= (1 << 63) else h


def run_case(name):
    sys.path.insert(0, REPO)
    sys.path.insert(0, "/root/reference/pkg/src")
    import fsefill  # noqa: F401
    from fsefill import fse
    from fsefill.fse import FseParams, weight_plane
    from fsefill.grid import build_grid

    from oracle import oracle as O
    from paper_2207_00233_b200 import synth

    fse._BACKENDS["compiled"] = O.ref_kernel()
    fse.set_backend("compiled")
    conceal_mod = sys.modules["fsefill.conceal"]
    record = {}
    cfg, frame, crop, kw, F = CASES[name]
    img, mask = synth.config_scene(cfg, frame)
    if crop is not None:
        r0, r1, c0, c1 = crop
        img, mask = img[r0:r1, c0:c1].copy(), mask[r0:r1, c0:c1].copy()
    p = FseParams(**kw)
    g = build_grid(img.shape[1], img.shape[0], p.block_size)

    def extrapolate_padded(win, params):
        values = np.ascontiguousarray(win.values, dtype=np.float64)
        w = weight_plane(values.shape, win.cls, params)
        if not (w > 0.0).any():
            raise fse.DegenerateWindowError("window has no usable samples")
        m, n = values.shape
        F1, F2 = (m, n) if F is None else F
        vp = np.zeros((F1, F2))
        wp = np.zeros((F1, F2))
        vp[:m, :n] = values
        wp[:m, :n] = w
        coeff, picks, _, _ = fse._BACKENDS["compiled"].run_fse(vp, wp, params.iterations, params.gamma)
        syn = (np.fft.ifft2(coeff) * (F1 * F2)).real[:m, :n]
        br0, br1, bc0, bc1 = win.block_rect
        b = ((win.origin[0] + br0) // p.block_size) * g.cols + (win.origin[1] + bc0) // p.block_size
        record[b] = O.canonical_picks(picks, (F1, F2))
        return syn[br0:br1, bc0:bc1].copy()

    conceal_mod.extrapolate_block = extrapolate_padded
    o_img, o_mask, rep = conceal_mod.conceal(img.astype(np.float64), mask, p, "optimized")
    lost = mask == 1
    keys = sorted(record)
    out = {
        "config": np.array(cfg), "frame": np.array(frame),
        "crop": np.array(crop if crop is not None else (0, 0, 0, 0)),
        "params": np.array([p.d, p.rho, p.delta, p.gamma, p.iterations, p.block_size]),
        "fft": np.array(F if F is not None else (0, 0)),
        "input_sums": np.array([int(img.astype(np.int64).sum()), int(mask.astype(np.int64).sum())]),
        "lost_values": o_img[lost],
        "out_mask_sum": np.array(int(o_mask.astype(np.int64).sum())),
        "batch_ptr": np.cumsum([0] + [len(b) for b in rep.batches]).astype(np.int32),
        "batch_blocks": np.asarray([b for bt in rep.batches for b in bt], dtype=np.int32),
        "unconcealed": np.asarray(rep.unconcealed_blocks, dtype=np.int32),
        "pick_blocks": np.asarray(keys, dtype=np.int32),
        "pick_hash": np.asarray([pick_hash(record[b]) for b in keys], dtype=np.int64),
        "sample_blocks": np.asarray(keys[::16], dtype=np.int32),
        "sample_picks": np.asarray([record[b] for b in keys[::16]], dtype=np.uint8),
    }
    np.savez_compressed(os.path.join(HERE, f"large_{name}.npz"), **out)
    return name, rep.blocks_processed, len(rep.batches), rep.wall_time


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    with get_context("spawn").Pool(len(names)) as pool:
        for r in pool.imap_unordered(run_case, names):
            print(*r, flush=True)
