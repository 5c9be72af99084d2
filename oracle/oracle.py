"""ORACLE — CPU restatement of the reference FSE path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this module.  The product package
(``paper_2207_00233_b200``) never does, and never falls back to it.

What is restated here (each function cites the reference lines it follows):

* ``run_fse``            -> ``fsefill._kernel.run_fse`` (``_kernel.pyx:128-187``) via
                            ``oracle/fse_oracle.c``, or the reference's own compiled
                            kernel from ``oracle/_ref`` when it was built here.
* ``weight_plane``       -> ``fse.py:105-119``
* grid helpers           -> ``grid.py:81-144``
* scheduler              -> ``schedule.py:28-105``
* ``conceal``            -> ``conceal.py:45-181`` (snapshot-per-batch, write-back,
                            deferred retry sweeps)
* ``extrapolate_block``  -> ``fse.py:142-176`` plus the FFT-size adapter of
                            SURVEY.md §8(c): values/weights zero-padded at the
                            top-left to F1 x F2, which is exactly the F-point FSE.

Parity is pinned by ``tests/golden/*.npz`` (generated from the reference itself by
``tests/golden/make_golden.py``) and by ``tests/test_oracle.py``.
"""

from __future__ import annotations

import ctypes
import glob
import os
import subprocess
import time
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

KNOWN, LOST, RECONSTRUCTED = 0, 1, 2          # image.py:14-16
AREA_A, AREA_BI, AREA_BO, AREA_R = 0, 1, 2, 3  # grid.py:20-23

# --------------------------------------------------------------------- kernels

_C_LIB = None


def build_c_oracle() -> str:
    """Compile oracle/fse_oracle.c -> oracle/libfse_oracle.so (no FMA contraction)."""
    src = os.path.join(HERE, "fse_oracle.c")
    out = os.path.join(HERE, "libfse_oracle.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", src, "-o", out, "-lm"]
        )
    return out


def _c_lib():
    global _C_LIB
    if _C_LIB is None:
        lib = ctypes.CDLL(build_c_oracle())
        d = ctypes.POINTER(ctypes.c_double)
        lib.oracle_run_fse.argtypes = [
            ctypes.c_int, ctypes.c_int, d, d, ctypes.c_int, ctypes.c_double,
            d, d, ctypes.POINTER(ctypes.c_int32), d, d,
        ]
        lib.oracle_run_fse.restype = ctypes.c_int
        _C_LIB = lib
    return _C_LIB


def _ptr(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t))


def run_fse_c(values, weights, iterations, gamma):
    """C restatement of run_fse; same contract as _kernel_py.py:13-30."""
    values = np.ascontiguousarray(values, dtype=np.float64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    m, n = values.shape
    c_re = np.empty((m, n)); c_im = np.empty((m, n))
    picks = np.empty((iterations, 2), dtype=np.int32)
    energies = np.empty(iterations + 1)
    residual = np.empty((m, n))
    rc = _c_lib().oracle_run_fse(
        m, n, _ptr(values), _ptr(weights), int(iterations), float(gamma),
        _ptr(c_re), _ptr(c_im), _ptr(picks, ctypes.c_int32), _ptr(energies), _ptr(residual),
    )
    if rc != 0:
        raise ValueError(f"oracle_run_fse failed: {rc}")
    return c_re + 1j * c_im, picks, energies, residual


_REF_KERNEL = None


def ref_kernel():
    """The reference's own compiled kernel (oracle/_ref, built by build_ref.sh), or None."""
    global _REF_KERNEL
    if _REF_KERNEL is None:
        hits = glob.glob(os.path.join(HERE, "_ref", "_kernel*.so"))
        if not hits:
            return None
        import importlib.util

        spec = importlib.util.spec_from_file_location("_kernel", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF_KERNEL = mod
    return _REF_KERNEL


def run_fse(values, weights, iterations, gamma, kernel="auto"):
    """kernel: 'ref' (oracle/_ref compiled reference), 'c' (restatement) or 'auto'."""
    if kernel in ("ref", "auto"):
        k = ref_kernel()
        if k is not None:
            return k.run_fse(values, weights, int(iterations), float(gamma))
        if kernel == "ref":
            raise RuntimeError("oracle/_ref not built (run oracle/build_ref.sh here)")
    return run_fse_c(values, weights, iterations, gamma)


def canonical_picks(picks, shape):
    """Fold each pick onto the lexicographically smaller member of its conjugate
    pair (the comparison rule of reference tests/reference.py:59-71)."""
    m, n = shape
    return [min((int(a), int(b)), ((m - int(a)) % m, (n - int(b)) % n)) for a, b in picks]


# ------------------------------------------------------------------- params

@dataclass(frozen=True)
class Params:
    """FseParams (fse.py:55-86) plus the FFT size (None = window size)."""
    d: int = 16
    rho: float = 0.8
    delta: float = 0.2
    gamma: float = 0.5
    iterations: int = 200
    block_size: int = 16
    fft_size: tuple | None = None


def weight_plane(shape, cls, rho, delta):
    """fse.py:105-119: rho^dist on A, delta*rho^dist on R, 0 on BI/BO; distance
    from the geometric centre ((M-1)/2, (N-1)/2) of the (possibly clipped) window."""
    m, n = shape
    ym = np.arange(m, dtype=np.float64) - (m - 1) / 2.0
    xn = np.arange(n, dtype=np.float64) - (n - 1) / 2.0
    decay = rho ** np.sqrt(ym[:, None] ** 2 + xn[None, :] ** 2)
    out = np.zeros(shape, dtype=np.float64)
    a = cls == AREA_A
    r = cls == AREA_R
    out[a] = decay[a]
    out[r] = delta * decay[r]
    return out


# --------------------------------------------------------------------- grid

@dataclass(frozen=True)
class Grid:
    """grid.py:26-88 — ceil block grid with ragged right/bottom blocks."""
    B: int
    rows: int
    cols: int
    H: int
    W: int

    @staticmethod
    def of(H, W, B):
        return Grid(B, -(-H // B), -(-W // B), H, W)

    def bounds(self, b):
        r, c = divmod(b, self.cols)
        return r * self.B, min(r * self.B + self.B, self.H), c * self.B, min(c * self.B + self.B, self.W)

    def neighbours(self, b):
        """grid.py:91-105 — 8-connected, row-major."""
        r, c = divmod(b, self.cols)
        out = []
        for rr in (r - 1, r, r + 1):
            if 0 <= rr < self.rows:
                for cc in (c - 1, c, c + 1):
                    if (rr, cc) != (r, c) and 0 <= cc < self.cols:
                        out.append(rr * self.cols + cc)
        return out


def lost_per_block(grid: Grid, mask):
    """grid.py:138-144."""
    pad = np.zeros((grid.rows * grid.B, grid.cols * grid.B), dtype=np.int64)
    pad[: grid.H, : grid.W] = mask == LOST
    return pad.reshape(grid.rows, grid.B, grid.cols, grid.B).sum(axis=(1, 3))


def classify(grid: Grid, mask, b, d):
    """grid.py:108-135 — window = block +- d clipped; returns (origin, cls, block_rect)."""
    r0, r1, c0, c1 = grid.bounds(b)
    wr0, wc0 = max(0, r0 - d), max(0, c0 - d)
    wr1, wc1 = min(grid.H, r1 + d), min(grid.W, c1 + d)
    sub = mask[wr0:wr1, wc0:wc1]
    cls = np.where(sub == RECONSTRUCTED, AREA_R, AREA_A).astype(np.uint8)
    inside = np.zeros(sub.shape, dtype=bool)
    inside[r0 - wr0 : r1 - wr0, c0 - wc0 : c1 - wc0] = True
    lost = sub == LOST
    cls[lost & inside] = AREA_BI
    cls[lost & ~inside] = AREA_BO
    return (wr0, wc0), cls, (r0 - wr0, r1 - wr0, c0 - wc0, c1 - wc0)


# ---------------------------------------------------------------- scheduler

def init_counts(grid: Grid, lossy_table):
    """schedule.py:28-57 — lossy 8-neighbour tally + rim bonus (+3 one edge,
    +5 two or more), -1 for blocks without loss."""
    lossy = np.asarray(lossy_table).reshape(grid.rows, grid.cols) > 0
    pad = np.pad(lossy.astype(np.int32), 1)
    cnt = sum(
        pad[1 + dr : 1 + dr + grid.rows, 1 + dc : 1 + dc + grid.cols]
        for dr in (-1, 0, 1) for dc in (-1, 0, 1) if (dr, dc) != (0, 0)
    ).astype(np.int32)
    er = (np.arange(grid.rows) == 0).astype(np.int32) + (np.arange(grid.rows) == grid.rows - 1)
    ec = (np.arange(grid.cols) == 0).astype(np.int32) + (np.arange(grid.cols) == grid.cols - 1)
    edges = er[:, None] + ec[None, :]
    cnt = cnt + np.where(edges == 1, 3, np.where(edges >= 2, 5, 0))
    cnt[~lossy] = -1
    return cnt.reshape(-1).astype(np.int32)


def schedule_all(grid: Grid, counts):
    """schedule.py:60-105 — phases of the neighbour-count wavefront: N_min over
    pending blocks, row-major greedy non-adjacent pick, commit (-1, neighbours -1)."""
    counts = np.array(counts, dtype=np.int64, copy=True)
    phases = []
    while (counts >= 0).any():
        nmin = counts[counts >= 0].min()
        taken = set()
        batch = []
        for b in np.flatnonzero(counts == nmin):
            b = int(b)
            nb = grid.neighbours(b)
            if any(x in taken for x in nb):
                continue
            batch.append(b)
            taken.add(b)
        for b in batch:
            counts[b] = -1
            for x in grid.neighbours(b):
                counts[x] -= 1
        phases.append(batch)
    return phases


# ------------------------------------------------------------------ conceal

def extrapolate(values, cls, block_rect, p: Params, kernel="auto", want_picks=False):
    """fse.py:142-176 with the F adapter. Returns block values
    (or None when degenerate, fse.py:150-151), plus picks if asked."""
    w = weight_plane(values.shape, cls, p.rho, p.delta)
    if not (w > 0.0).any():
        return (None, None) if want_picks else None
    m, n = values.shape
    if p.fft_size is None:
        F1, F2 = m, n
    else:
        F1, F2 = p.fft_size
    vpad = np.zeros((F1, F2)); wpad = np.zeros((F1, F2))
    vpad[:m, :n] = values
    wpad[:m, :n] = w
    coeff, picks, _, _ = run_fse(vpad, wpad, p.iterations, p.gamma, kernel)
    syn = (np.fft.ifft2(coeff) * (F1 * F2)).real[:m, :n]
    r0, r1, c0, c1 = block_rect
    blk = syn[r0:r1, c0:c1].copy()
    return (blk, picks) if want_picks else blk


@dataclass
class Report:
    order: str
    blocks_processed: int
    wall_time: float
    batches: list = field(default_factory=list)
    unconcealed_blocks: list = field(default_factory=list)
    picks: dict = field(default_factory=dict)
    sched_time: float = 0.0   # seconds spent in schedule_all (inside wall_time)
    n_lossy: int = 0          # lossy blocks of the whole frame


def conceal(image, mask, p: Params, order="optimized", kernel="auto", want_picks=False,
            block_limit=None):
    """conceal.py:97-181.  optimized: every member of a phase is classified and
    snapshotted before any write-back; linescan: strictly sequential row-major.
    Degenerate windows are deferred to row-major retry sweeps (conceal.py:69-94).
    block_limit (bench sampling only) stops after that many fitted blocks."""
    if order not in ("optimized", "linescan"):
        raise ValueError(f"unknown order {order!r}")
    img = np.array(image, dtype=np.float64, copy=True)
    msk = np.array(mask, dtype=np.uint8, copy=True)
    grid = Grid.of(img.shape[0], img.shape[1], p.block_size)
    table = lost_per_block(grid, msk)
    t0 = time.perf_counter()
    picks_out = {}
    sched_time = 0.0
    batches, deferred = [], []
    processed = 0

    def snap(b):
        (wr, wc), cls, rect = classify(grid, msk, b, p.d)
        h, w = cls.shape
        return img[wr : wr + h, wc : wc + w].copy(), cls, rect

    def write(b, blk):
        r0, r1, c0, c1 = grid.bounds(b)
        lost = msk[r0:r1, c0:c1] == LOST
        img[r0:r1, c0:c1][lost] = blk[lost]
        msk[r0:r1, c0:c1][lost] = RECONSTRUCTED

    def fit(b, s):
        blk, pk = extrapolate(*s, p, kernel, want_picks=True)
        if pk is not None and want_picks:
            picks_out[b] = pk
        return blk

    if order == "linescan":
        for b in np.flatnonzero(table.reshape(-1) > 0):
            b = int(b)
            blk = fit(b, snap(b))
            if blk is None:
                deferred.append(b)
                continue
            write(b, blk)
            batches.append([b])
            processed += 1
            if block_limit and processed >= block_limit:
                break
    else:
        ts = time.perf_counter()
        phases = schedule_all(grid, init_counts(grid, table))
        sched_time = time.perf_counter() - ts
        for phase in phases:
            snaps = [snap(b) for b in phase]
            done = []
            for b, s in zip(phase, snaps):
                blk = fit(b, s)
                if blk is None:
                    deferred.append(b)
                    continue
                write(b, blk)
                done.append(b)
                processed += 1
            if done:
                batches.append(done)
            if block_limit and processed >= block_limit:
                break

    pending = sorted(deferred)
    for _ in range(max(grid.rows, grid.cols)):
        if not pending:
            break
        still = []
        for b in pending:
            blk = fit(b, snap(b))
            if blk is None:
                still.append(b)
            else:
                write(b, blk)
                batches.append([b])
                processed += 1
        if len(still) == len(pending):
            break
        pending = still
    rep = Report(order, processed, time.perf_counter() - t0, batches, pending, picks_out,
                 sched_time, int((table > 0).sum()))
    return img, msk, rep
