"""Streaming concealment of a frame sequence (video): SURVEY.md §8(f) rank 4.

The reference conceals one image per call (fsefill/conceal.py:97-181); a video
use case calls it frame after frame.  ``ConcealStream`` keeps the
GPU busy across frames instead: frames are pushed one at a time, gathered into
batches, and each batch runs through a pipeline whose stages overlap with the
neighbouring batches' --

    host:   copy into a pinned slot -> plan (C++ threads)
    up:     upload batch k+1
    down:   download batch k-1 (waits only for batch k-1's levels)
    main:   levels of batch k (every frame's level l in one launch)

Uploads and downloads use separate streams: on one in-order copy stream the
next batch's upload would queue behind the previous batch's download, which
waits for that batch's levels, and the GPU would idle between batches.

A background thread plans and enqueues batches in order, so ``push`` returns
at once; concealed frames come back in push order, from ``push`` (whatever has
finished) and ``flush`` (everything).  Each frame's result is exactly
``conceal(frame, mask, params, order, precision=...)`` (tested).
"""

from __future__ import annotations

import queue
import threading

import numpy as np

from .conceal import (OPTIMIZED, ORDERS, PRECISIONS, balance_batch, balance_for_device, build_plans,
                      run_frames_device)
from .fse import FseParams


class ConcealStream:
    """Conceal frames of one shape as they arrive.

    params/order/precision as in ``conceal``; ``batch`` frames share a launch
    sequence (more = wider levels, more latency); ``depth`` batches may be in
    flight (pinned host slots and device buffers are allocated once).
    """

    def __init__(self, params: FseParams | None, shape, batch: int = 16, precision: str = "fp64",
                 order: str = OPTIMIZED, depth: int = 3, plan_threads: int = 0, in_dtype=np.uint8):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("ConcealStream needs a CUDA device (no CPU fallback)")
        if order not in ORDERS:
            raise ValueError(f"unknown order {order!r}")
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        if batch < 1 or depth < 1:
            raise ValueError("batch and depth must be >= 1")
        self.params = params if params is not None else FseParams()
        self.order, self.precision, self.batch, self.plan_threads = order, precision, batch, plan_threads
        H, W = (int(x) for x in shape)
        self.shape = (H, W)
        self._torch = torch
        tdt = torch.float64 if precision == "fp64" else torch.float32
        self._tdt = tdt
        # frames travel in their own dtype (uint8 video: 1 B/sample over PCIe)
        # and are widened on the device
        self._in_np = np.dtype(in_dtype)
        itd = torch.from_numpy(np.zeros(1, dtype=self._in_np)).dtype
        self.device = torch.cuda.current_device()
        self._main = torch.cuda.Stream(device=self.device)
        self._up = torch.cuda.Stream(device=self.device)
        self._down = torch.cuda.Stream(device=self.device)
        # slot = pinned inputs + outputs on the host, frames + masks on the device
        self._slots = []
        for _ in range(depth):
            self._slots.append(dict(
                img_h=torch.empty((batch, H, W), dtype=itd, pin_memory=True),
                in_d=torch.empty((batch, H, W), dtype=itd, device=self.device) if itd != tdt else None,
                msk_h=torch.empty((batch, H, W), dtype=torch.uint8, pin_memory=True),
                img_d=torch.empty((batch, H, W), dtype=tdt, device=self.device),
                msk_d=torch.empty((batch, H, W), dtype=torch.uint8, device=self.device),
                omsk_d=torch.empty((batch, H, W), dtype=torch.uint8, device=self.device),
                done=None, n=0))
        self._free = queue.Queue()
        for i in range(depth):
            self._free.put(i)
        self._pending = []       # results collected while waiting for a free slot
        self._fill = None        # slot being filled by push
        self._inflight = []      # slots submitted, in order
        self._work = queue.Queue()
        self._err = None
        self._worker = threading.Thread(target=self._run, daemon=True)
        self._worker.start()

    # ---------------------------------------------------------------- worker
    def _run(self):
        torch = self._torch
        torch.cuda.set_device(self.device)
        while True:
            item = self._work.get()
            if item is None:
                return
            i = item
            s = self._slots[i]
            n = s["n"]
            try:
                with torch.cuda.stream(self._up):  # upload (pinned -> device), widen
                    if s["in_d"] is None:
                        s["img_d"][:n].copy_(s["img_h"][:n], non_blocking=True)
                    else:
                        s["in_d"][:n].copy_(s["img_h"][:n], non_blocking=True)
                        s["img_d"][:n].copy_(s["in_d"][:n])
                    s["msk_d"][:n].copy_(s["msk_h"][:n], non_blocking=True)
                    up = self._up.record_event()
                plans = build_plans(list(s["msk_h"][:n].numpy()), self.params, self.order, self.plan_threads)
                if n == 1:
                    balance_for_device(plans[0], self.params, self.precision)
                else:
                    balance_batch(plans, self.params, self.precision)
                self._main.wait_event(up)
                with torch.cuda.stream(self._main):
                    run_frames_device(plans, list(s["img_d"][:n]), list(s["msk_d"][:n]),
                                      list(s["omsk_d"][:n]), self.params, self.precision,
                                      stream=self._main.cuda_stream)
                    ran = self._main.record_event()
                # results land in fresh pinned buffers that are handed to the
                # caller as they are (no host copy; torch's pinned caching
                # allocator recycles them once the caller drops the frames)
                s["out_h"] = torch.empty((n,) + self.shape, dtype=self._tdt, pin_memory=True)
                s["omsk_h"] = torch.empty((n,) + self.shape, dtype=torch.uint8, pin_memory=True)
                with torch.cuda.stream(self._down):  # download (device -> pinned)
                    self._down.wait_event(ran)
                    s["out_h"][:n].copy_(s["img_d"][:n], non_blocking=True)
                    s["omsk_h"][:n].copy_(s["omsk_d"][:n], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(self._down)
                s["plans"] = plans  # keep the plans alive until the batch is done
                s["done"] = ev
            except Exception as e:  # surfaced to the caller on the next push/flush
                self._err = e
                s["done"] = "error"

    # ------------------------------------------------------------------ API
    def push(self, image, mask) -> list:
        """Queue one frame; returns the (image, mask) results that have finished
        since the last call, in push order."""
        self._check()
        if np.shape(image) != self.shape or np.shape(mask) != self.shape:
            raise ValueError(f"frames of this stream are {self.shape}")
        if self._fill is None:
            self._fill = self._acquire()
        s = self._slots[self._fill]
        k = s["n"]
        s["img_h"][k].numpy()[...] = image
        s["msk_h"][k].numpy()[...] = np.asarray(mask, dtype=np.uint8)
        s["n"] = k + 1
        if s["n"] == self.batch:
            self._submit()
        return self._collect(block=False)

    def flush(self) -> list:
        """Submit the partial batch and return every remaining result, in order."""
        self._check()
        if self._fill is not None and self._slots[self._fill]["n"] > 0:
            self._submit()
        return self._collect(block=True)

    def close(self) -> None:
        if self._worker.is_alive():
            self._work.put(None)
            self._worker.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -------------------------------------------------------------- internals
    def _check(self):
        if self._err is not None:
            raise self._err

    def _submit(self):
        i = self._fill
        self._fill = None
        self._slots[i]["done"] = None
        self._inflight.append(i)
        self._work.put(i)

    def _acquire(self) -> int:
        while self._free.empty():
            # backpressure: every slot is in flight -- wait for the oldest
            self._pending.extend(self._collect_one(block=True))
        return self._free.get()

    def _collect_one(self, block: bool) -> list:
        if not self._inflight:
            return []
        i = self._inflight[0]
        s = self._slots[i]
        while s["done"] is None:  # the worker has not enqueued it yet
            if not block:
                return []
            threading.Event().wait(0.0005)
        if s["done"] == "error":
            self._check()
        if not block and not s["done"].query():
            return []
        s["done"].synchronize()
        n = s["n"]
        oi, om = s["out_h"].numpy(), s["omsk_h"].numpy()
        out = [(oi[f], om[f]) for f in range(n)]
        s["n"] = 0
        s["plans"] = s["out_h"] = s["omsk_h"] = None
        self._inflight.pop(0)
        self._free.put(i)
        return out

    def _collect(self, block: bool) -> list:
        res, self._pending = self._pending, []
        while self._inflight:
            got = self._collect_one(block)
            if not got and not block:
                break
            res.extend(got)
        return res
