"""Neighbour-count wavefront order (API mirror of fsefill.schedule).

``init_counts`` and ``schedule_all`` run in the C++ scheduler of libfse_b200
(csrc/fse_plan.cpp, a bucket queue over count values); they reproduce
schedule.py:28-57 and :97-105 of the reference exactly.  ``select_batch`` /
``commit_batch`` are the single-step forms of the same rules (schedule.py:60-94),
kept for API compatibility.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .grid import BlockGrid, neighbors

Batch = list


class EmptyScheduleError(RuntimeError):
    """A batch was requested while no block is pending (schedule.py:24-25)."""


def init_counts(grid: BlockGrid, lost_counts) -> np.ndarray:
    """Lossy-neighbour tally + rim bonus (+3 / +5); -1 for blocks without loss."""
    lossy = np.ascontiguousarray((np.asarray(lost_counts).reshape(grid.rows, grid.cols) > 0)
                                 .astype(np.uint8))
    counts = np.empty(grid.rows * grid.cols, dtype=np.int32)
    _lib.check(_lib.lib().fse_init_counts(lossy.ctypes.data, grid.rows, grid.cols,
                                          _lib.ptr32(counts)))
    return counts


def select_batch(grid: BlockGrid, counts) -> list:
    """Pending blocks with the minimum count, row-major, skipping neighbours of
    blocks already taken for this batch (schedule.py:60-82)."""
    counts = np.asarray(counts)
    pending = counts >= 0
    if not pending.any():
        raise EmptyScheduleError("no blocks awaiting concealment")
    n_min = int(counts[pending].min())
    taken = set()
    batch = []
    for b in np.flatnonzero(counts == n_min).tolist():
        if taken.isdisjoint(neighbors(grid, b)):
            batch.append(b)
            taken.add(b)
    return batch


def commit_batch(grid: BlockGrid, counts: np.ndarray, batch) -> None:
    """Members go to -1, every neighbour count drops by one (schedule.py:85-94)."""
    for b in batch:
        counts[b] = -1
        for nb in neighbors(grid, b):
            counts[nb] -= 1


def schedule_all(grid: BlockGrid, counts) -> list:
    """Full batch sequence from an initial count state (input not modified)."""
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.int32).reshape(-1))
    n_pending = int((c >= 0).sum())
    ptr = np.zeros(n_pending + 1, dtype=np.int32)
    blocks = np.zeros(max(n_pending, 1), dtype=np.int32)
    nb = np.zeros(1, dtype=np.int32)
    _lib.check(_lib.lib().fse_schedule_all(_lib.ptr32(c), grid.rows, grid.cols, _lib.ptr32(ptr),
                                           _lib.ptr32(blocks), _lib.ptr32(nb)))
    k = int(nb[0])
    return [blocks[ptr[i]:ptr[i + 1]].tolist() for i in range(k)]


def render_batch_trace(grid: BlockGrid, batches) -> str:
    """1-based batch number per block, -1 for untouched blocks (schedule.py:108-116)."""
    stamp = np.full(grid.n_blocks, -1, dtype=np.int64)
    for i, batch in enumerate(batches, start=1):
        stamp[list(batch)] = i
    return "\n".join(" ".join(map(str, row)) for row in stamp.reshape(grid.rows, grid.cols).tolist())
