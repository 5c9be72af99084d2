"""Seeded synthetic frames and loss masks for the BASELINE.json configurations.

The reference measures on the paper's photographs, which are not
available; BASELINE.json fixes seeded synthetic stand-ins instead.  The ranges
BASELINE leaves open are fixed here, once:

* image  = 128 + sum of ``n_sin`` plane sinusoids (amplitude U(10, 40),
  orientation U(0, pi), frequency U(0.005, 0.08) cycles/px, phase U(0, 2 pi))
  + ``n_poly`` star-shaped random polygons (3-8 vertices, radius U(0.05, 0.25) of
  the short side, constant offset U(-60, 60)) + Gaussian noise sigma = 2,
  clipped to [0, 255] and rounded to uint8.
* masks live on a 16 x 16 loss-cell grid (``ceil`` at ragged edges) and mark
  whole cells LOST:
  ``isolated`` i.i.d. Bernoulli cells (optionally excluding the rim cells),
  ``hburst`` horizontal runs, ``burst2d`` runs in both directions,
  ``mixed`` half bursts / half isolated cells.
* seeds: config c -> image 1000 + c, mask 2000 + c; config 4 frame f ->
  image 4000 + f, mask 5000 + f.
"""

from __future__ import annotations

import numpy as np

KNOWN, LOST = np.uint8(0), np.uint8(1)
CELL = 16


def synthetic_frame(h: int, w: int, seed: int, n_sin: int = 8, n_poly: int = 6) -> np.ndarray:
    rng = np.random.default_rng(seed)
    y = np.arange(h, dtype=np.float64)
    x = np.arange(w, dtype=np.float64)
    img = np.full((h, w), 128.0)
    for _ in range(n_sin):
        amp = rng.uniform(10.0, 40.0)
        th = rng.uniform(0.0, np.pi)
        f = rng.uniform(0.005, 0.08)
        ph = rng.uniform(0.0, 2.0 * np.pi)
        ax = 2.0 * np.pi * f * np.cos(th) * x
        by = 2.0 * np.pi * f * np.sin(th) * y + ph
        # sin(ax + by) = sin(ax) cos(by) + cos(ax) sin(by): two outer products
        img += amp * (np.outer(np.cos(by), np.sin(ax)) + np.outer(np.sin(by), np.cos(ax)))
    short = min(h, w)
    for _ in range(n_poly):
        nv = int(rng.integers(3, 9))
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        rad = rng.uniform(0.05, 0.25) * short * rng.uniform(0.6, 1.0, nv)
        ang = np.sort(rng.uniform(0.0, 2.0 * np.pi, nv))
        vy = cy + rad * np.sin(ang)
        vx = cx + rad * np.cos(ang)
        off = rng.uniform(-60.0, 60.0)
        r0, r1 = max(0, int(np.floor(vy.min()))), min(h, int(np.ceil(vy.max())) + 1)
        c0, c1 = max(0, int(np.floor(vx.min()))), min(w, int(np.ceil(vx.max())) + 1)
        if r0 >= r1 or c0 >= c1:
            continue
        py = np.arange(r0, r1, dtype=np.float64)[:, None] + 0.5
        px = np.arange(c0, c1, dtype=np.float64)[None, :] + 0.5
        inside = np.zeros((r1 - r0, c1 - c0), dtype=bool)
        for i in range(nv):  # even-odd crossing rule
            y0, x0, y1, x1 = vy[i], vx[i], vy[(i + 1) % nv], vx[(i + 1) % nv]
            if y0 == y1:
                continue
            cond = (py >= min(y0, y1)) & (py < max(y0, y1))
            xc = x0 + (py - y0) * (x1 - x0) / (y1 - y0)
            inside ^= cond & (px < xc)
        img[r0:r1, c0:c1] += off * inside
    img += rng.normal(0.0, 2.0, (h, w))
    return np.floor(np.clip(img, 0.0, 255.0) + 0.5).astype(np.uint8)


def _cells(h, w):
    return -(-h // CELL), -(-w // CELL)


def _paint(h, w, lost_cells):
    cr, cc = _cells(h, w)
    mask = np.repeat(np.repeat(lost_cells.astype(np.uint8), CELL, 0), CELL, 1)[:h, :w]
    return np.where(mask > 0, LOST, KNOWN).astype(np.uint8)


def _bursts(rng, cells, target, lo, hi, dirs):
    cr, cc = cells.shape
    goal = int(round(target * cr * cc))
    guard = 0
    while cells.sum() < goal and guard < 100 * cr * cc:
        guard += 1
        L = int(rng.integers(lo, hi + 1))
        d = dirs[int(rng.integers(0, len(dirs)))]
        if d == "h":
            r, c = int(rng.integers(0, cr)), int(rng.integers(0, max(1, cc - L + 1)))
            cells[r, c : c + L] = True
        else:
            r, c = int(rng.integers(0, max(1, cr - L + 1))), int(rng.integers(0, cc))
            cells[r : r + L, c] = True
    return cells


def loss_mask(h: int, w: int, kind: str, fraction: float, seed: int,
              exclude_rim: bool = False) -> np.ndarray:
    rng = np.random.default_rng(seed)
    cr, cc = _cells(h, w)
    cells = np.zeros((cr, cc), dtype=bool)
    if kind == "isolated":
        cells = rng.uniform(size=(cr, cc)) < fraction
        if exclude_rim:
            cells[0, :] = cells[-1, :] = False
            cells[:, 0] = cells[:, -1] = False
    elif kind == "hburst":
        cells = _bursts(rng, cells, fraction, 2, 6, ("h",))
    elif kind == "burst2d":
        cells = _bursts(rng, cells, fraction, 2, 8, ("h", "v"))
    elif kind == "mixed":
        cells = _bursts(rng, cells, fraction / 2, 2, 6, ("h", "v"))
        free = ~cells
        add = rng.uniform(size=(cr, cc)) < (fraction / 2) / max(1e-9, free.mean())
        cells |= add & free
    else:
        raise ValueError(f"unknown mask kind {kind!r}")
    return _paint(h, w, cells)


# BASELINE.json configs -> (H, W, n_sin, n_poly, mask kind, fraction, rim excluded)
CONFIGS = {
    1: (512, 512, 8, 6, "isolated", 0.10, True),
    2: (512, 512, 8, 6, "hburst", 0.20, False),
    3: (1080, 1920, 16, 12, "isolated", 0.30, False),
    4: (1080, 1920, 16, 12, "mixed", 0.20, False),
    5: (2160, 3840, 16, 12, "burst2d", 0.50, False),
}


def config_scene(config: int, frame: int = 0):
    """(image uint8, mask uint8) for a BASELINE config (frame only for config 4)."""
    h, w, ns, npoly, kind, frac, rim = CONFIGS[config]
    if config == 4:
        iseed, mseed = 4000 + frame, 5000 + frame
    else:
        iseed, mseed = 1000 + config, 2000 + config
    img = synthetic_frame(h, w, iseed, ns, npoly)
    mask = loss_mask(h, w, kind, frac, mseed, exclude_rim=rim)
    return img, mask
