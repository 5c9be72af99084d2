"""Reporting harness of the concealment path: PSNR over
the non-KNOWN samples, the order/block-size sweep and its CSV, mirroring
fsefill.evalkit (/root/reference/pkg/src/fsefill/evalkit.py:67-160).

``psnr`` and ``write_csv`` are host-side formatting of results; ``bench`` runs
every configuration through this package's ``conceal`` (the sm_100a path).  The
reference's ``threads`` sweep is kept for the row layout: a B200 run does not
depend on host threads, so every thread count reports the same concealment
(its own timing), and ``speedup`` is measured against the one-thread row of the
same order and block size, as in the reference.  On the device the PSNR sums
come from ``fse_quantize_psnr`` (conceal.quantize_psnr_device) instead.
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass, replace

import numpy as np

from .conceal import LINESCAN, OPTIMIZED, conceal
from .fse import FseParams

KNOWN, LOST = 0, 1


def psnr(original: np.ndarray, result: np.ndarray, mask: np.ndarray) -> float:
    """evalkit.py:67-81: peak SNR (peak 255) over the samples mask marks
    non-KNOWN; +inf for identical signals, ValueError for an empty region."""
    region = np.asarray(mask) != KNOWN
    if not region.any():
        raise ValueError("mask selects no samples to compare")
    d = np.asarray(original, dtype=np.float64)[region] - np.asarray(result, dtype=np.float64)[region]
    mse = float(np.mean(d * d))
    if mse == 0.0:
        return float("inf")
    return 10.0 * np.log10(255.0 ** 2 / mse)


@dataclass(frozen=True)
class BenchRow:
    """evalkit.py:84-91."""

    order: str
    block_size: int
    threads: int
    psnr_db: float
    seconds: float
    speedup: float


def bench(image, mask, *, block_sizes=(16,), threads=(1,), orders=(LINESCAN, OPTIMIZED),
          params: FseParams | None = None, repeats: int = 1, precision: str = "fp64") -> list:
    """evalkit.py:94-148 on the GPU path: lost samples are zeroed first, the
    fastest of `repeats` runs is kept, linescan appears at one thread only,
    speedup is against the one-thread run of the same order and block size."""
    if params is None:
        params = FseParams()
    damaged = np.array(image, dtype=np.float64, copy=True)
    damaged[np.asarray(mask) == LOST] = 0.0
    rows = []
    for block_size in block_sizes:
        p = replace(params, block_size=block_size)
        for order in orders:
            thread_list = [1] if order == LINESCAN else sorted(set(threads) | {1})
            base = None
            for t in thread_list:
                best, result = None, None
                for _ in range(max(1, repeats)):
                    out, _, rep = conceal(damaged, mask, p, order=order, threads=t, precision=precision)
                    if best is None or rep.wall_time < best:
                        best, result = rep.wall_time, out
                if t == 1:
                    base = best
                rows.append(BenchRow(order=order, block_size=block_size, threads=t,
                                     psnr_db=psnr(image, result, mask), seconds=best, speedup=base / best))
    return rows


CSV_HEADER = "order,block_size,threads,psnr_db,seconds,speedup"


def write_csv(rows, out: io.TextIOBase) -> None:
    """evalkit.py:151-160: header, then one row per configuration with
    psnr/seconds to 6 decimals and speedup to 3."""
    w = csv.writer(out, lineterminator="\n")
    w.writerow(CSV_HEADER.split(","))
    for r in rows:
        w.writerow([r.order, r.block_size, r.threads, f"{r.psnr_db:.6f}", f"{r.seconds:.6f}",
                    f"{r.speedup:.3f}"])


__all__ = ["psnr", "BenchRow", "bench", "CSV_HEADER", "write_csv", "OPTIMIZED", "LINESCAN"]
