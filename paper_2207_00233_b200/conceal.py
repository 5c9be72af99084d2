"""End-to-end concealment on a B200 (drop-in for fsefill.conceal.conceal).

``conceal(image, mask, params, order, threads)`` keeps the reference's contract
(/root/reference/pkg/src/fsefill/conceal.py:97-181): same arguments, same
ValueErrors, inputs untouched, returns (image float64, mask uint8,
ConcealReport) with the reference's batches / blocks_processed /
unconcealed_blocks.  ``precision`` ("fp64" default, or "fp32") is added, and
FseParams gains ``fft_size``.

How it runs:
  1. C++ plan (csrc/fse_plan.cpp): the reference batches, effective ranks with
     host-decided deferral/retry sweeps, and dependency levels.
  2. One device launch per level (csrc/fse_kernel.cuh, MODE 0): each CTA
     classifies its window from the original mask + ranks, builds weights,
     fits the model and writes its block's LOST samples back into the image.
  3. A mask pass marks concealed samples RECONSTRUCTED.
``conceal_batch`` does the same for many equally sized frames with all frames'
levels merged into one launch each (frame-parallel, BASELINE config 4).
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .fse import FseParams, PRECISIONS, decay_table

LINESCAN = "linescan"
OPTIMIZED = "optimized"
ORDERS = (LINESCAN, OPTIMIZED)


@dataclass
class ConcealReport:
    """conceal.py:35-42."""

    order: str
    threads: int
    blocks_processed: int
    wall_time: float
    batches: list = field(default_factory=list)
    unconcealed_blocks: list = field(default_factory=list)
    levels: int = 0  # dependency levels launched (B200 addition)


class Plan:
    """Owner of an FsePlan* (C++ scheduler result)."""

    def __init__(self, handle: int):
        self.handle = ctypes.c_void_p(handle)
        s = np.zeros(10, dtype=np.int32)
        _lib.check(_lib.lib().fse_plan_sizes(self.handle, _lib.ptr32(s)))
        (self.rows, self.cols, self.n_lossy, self.n_processed, self.n_batches, self.n_entries,
         self.n_levels, self.n_unconcealed, self.max_wr, self.max_wc) = (int(x) for x in s)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.lib().fse_plan_free(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self.handle = None

    def _csr(self, fn, n, m):
        ptr = np.zeros(n + 1, dtype=np.int32)
        blocks = np.zeros(max(m, 1), dtype=np.int32)
        _lib.check(fn(self.handle, _lib.ptr32(ptr), _lib.ptr32(blocks)))
        return [blocks[ptr[i]:ptr[i + 1]].tolist() for i in range(n)]

    def batches(self) -> list:
        return self._csr(_lib.lib().fse_plan_batches, self.n_batches, self.n_entries)

    def levels(self) -> list:
        return self._csr(_lib.lib().fse_plan_levels, self.n_levels, self.n_processed)

    def rebalance(self, narrow: int, wave: int = 0) -> int:
        """Level balancing (fse_plan_rebalance): blocks with slack move from levels
        wider than ``narrow`` windows into later levels with free slots.  Ranks,
        batches and results are unchanged.  Returns the number of moved blocks."""
        moved = np.zeros(1, dtype=np.int32)
        _lib.check(_lib.lib().fse_plan_rebalance(self.handle, int(narrow), int(wave), _lib.ptr32(moved)))
        return int(moved[0])

    def ranks(self) -> np.ndarray:
        r = np.zeros(self.rows * self.cols, dtype=np.int32)
        _lib.check(_lib.lib().fse_plan_ranks(self.handle, _lib.ptr32(r)))
        return r

    def to_bytes(self) -> bytes:
        """The plan serialised (fse_plan_export): broadcast it instead of planning
        the same frame on every rank."""
        n = int(_lib.lib().fse_plan_export_size(self.handle))
        if n < 0:
            _lib.check(n)
        buf = (ctypes.c_ubyte * n)()
        _lib.check(_lib.lib().fse_plan_export(self.handle, buf, n))
        return bytes(buf)

    @classmethod
    def from_bytes(cls, data) -> "Plan":
        """A plan from fse_plan_export's bytes (fse_plan_import)."""
        a = np.frombuffer(bytes(data), dtype=np.uint8)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().fse_plan_import(a.ctypes.data, a.size, ctypes.byref(h)))
        return cls(h.value)

    def unconcealed(self) -> list:
        u = np.zeros(max(self.n_unconcealed, 1), dtype=np.int32)
        _lib.check(_lib.lib().fse_plan_unconcealed(self.handle, _lib.ptr32(u)))
        return u[: self.n_unconcealed].tolist()


_SM_COUNT: dict = {}


def balance_for_device(plan: "Plan", params: FseParams, precision: str, frames: int = 1, world: int = 1) -> int:
    """Level balancing of a one-frame plan for the current CUDA device: narrow =
    the SM count (levels of at most that many windows run one window per SM, at
    a lone window's latency however few they are, so their free slots take
    blocks of the wide levels for nothing).  Plans of a multi-frame call are
    left alone: their levels merge across frames.  Levels of less than one wave
    (wave = SMs x resident CTAs per SM of the fast kernel) are filled up to the
    wave as well.  FSE_BALANCE=0 turns it off; FSE_BALANCE_WAVE=0 fills narrow
    levels only, =2 fills every level of at most one wave up to it (measured in
    DESIGN.md: 30.8 / 30.4 / 31.8 ms on config 3 for 0 / 1 / 2)."""
    if frames != 1 or os.environ.get("FSE_BALANCE", "1") == "0":
        return 0
    # the pass is sequential (1.3 ms on a 1080p frame at B = 4, 9 ms on a 4K one, 65 ms on a 4K frame at
    # B = 2, whose band-parallel plan itself takes 25 ms): skipped on the largest grids
    if plan.rows * plan.cols > int(os.environ.get("FSE_BALANCE_MAX_BLOCKS", "600000")):
        return 0
    import torch

    if not torch.cuda.is_available():
        return 0
    dev = torch.cuda.current_device()
    sms = _SM_COUNT.get(dev)
    if sms is None:
        sms = _SM_COUNT[dev] = torch.cuda.get_device_properties(dev).multi_processor_count
    F = params.fft_size if isinstance(params.fft_size, int) else 0
    per_sm = {("fp64", 64): 3, ("fp32", 64): 4, ("fp64", 32): 6, ("fp32", 32): 8,
              ("fp64", 128): 1, ("fp32", 128): 1}.get((precision, F), 0)
    mode = os.environ.get("FSE_BALANCE_WAVE", "1")
    wave = sms * per_sm if mode in ("1", "2") else 0
    # a frame sharded over `world` GPUs (strips) has that many times the slots per level
    sms, wave = sms * max(1, world), wave * max(1, world)
    if os.environ.get("FSE_BALANCE_NARROW"):  # tests: force moves on small frames
        sms, wave = int(os.environ["FSE_BALANCE_NARROW"]), 0
    return plan.rebalance(wave if mode == "2" and wave else sms, wave)


def balance_batch(plans, params: FseParams, precision: str) -> int:
    """Level balancing of the plans of one multi-frame session: the session's
    launches merge each level over the frames of a group (fse_set_groups), so
    each frame's share of a one-window-per-SM launch is SMs / frames per group.
    Plans are balanced on host threads (the C call releases the GIL).
    FSE_BALANCE_BATCH=0 turns it off."""
    n = len(plans)
    if n < 2 or os.environ.get("FSE_BALANCE", "1") == "0" or os.environ.get("FSE_BALANCE_BATCH", "1") == "0":
        return 0
    import torch

    if not torch.cuda.is_available():
        return 0
    dev = torch.cuda.current_device()
    sms = _SM_COUNT.get(dev)
    if sms is None:
        sms = _SM_COUNT[dev] = torch.cuda.get_device_properties(dev).multi_processor_count
    groups = max(1, min(int(os.environ.get("FSE_GROUPS", "2")), n))
    narrow = sms * groups // n
    if narrow < 2:
        return 0
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(n, max(1, (3 * len(os.sched_getaffinity(0))) // 4))) as ex:
        return sum(ex.map(lambda pl: pl.rebalance(narrow, 0), plans))


def _order_code(order: str) -> int:
    return _lib.FSE_ORDER_LINESCAN if order == LINESCAN else _lib.FSE_ORDER_OPTIMIZED


def build_plan(mask: np.ndarray, params: FseParams, order: str = OPTIMIZED, plan_threads: int = 0) -> Plan:
    """Host plan of one frame (fse_plan_build_threads; 0 = automatic thread count,
    1 = the sequential planner -- the plan is identical either way)."""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    h = ctypes.c_void_p()
    pc = params.to_c()
    _lib.check(_lib.lib().fse_plan_build_threads(m.ctypes.data, m.shape[0], m.shape[1], ctypes.byref(pc),
                                                 _order_code(order), int(plan_threads), ctypes.byref(h)))
    return Plan(h.value)


def build_plans(masks, params: FseParams, order: str = OPTIMIZED, threads: int = 0) -> list:
    ms = [np.ascontiguousarray(m, dtype=np.uint8) for m in masks]
    n = len(ms)
    if n == 0:
        return []
    H, W = ms[0].shape
    if any(m.shape != (H, W) for m in ms):
        raise ValueError("all masks of a batch must share one shape")
    arr = (ctypes.c_void_p * n)(*[m.ctypes.data for m in ms])
    out = (ctypes.c_void_p * n)()
    pc = params.to_c()
    _lib.check(_lib.lib().fse_plan_build_many(n, arr, H, W, ctypes.byref(pc), _order_code(order),
                                              int(threads), out))
    return [Plan(out[i]) for i in range(n)]


def _validate(image, mask, params, order, threads, precision):
    if params is None:
        params = FseParams()
    if order not in ORDERS:
        raise ValueError(f"unknown order {order!r}")
    if threads < 1:
        raise ValueError("threads must be >= 1")
    if order == LINESCAN and threads != 1:
        raise ValueError("linescan order is sequential; threads must be 1")
    if np.shape(mask) != np.shape(image):
        raise ValueError(f"mask shape {np.shape(mask)} != image shape {np.shape(image)}")
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    return params


class DeviceContext:
    """Device-resident constants shared by calls with the same params (the
    rho^dist table) plus the torch module handle."""

    _cache: dict = {}

    @classmethod
    def decay(cls, params: FseParams, dim: int):
        import torch

        # one table per device: a pointer from another device's memory would
        # reach the kernel of a call on this one
        key = (torch.cuda.current_device(), params.rho, dim)
        t = cls._cache.get(key)
        if t is None:
            t = torch.from_numpy(decay_table(params.rho, dim)).cuda()
            cls._cache[key] = t
        return t


def check_device_frames(images_dev, masks_dev, plans, precision: str, block_size: int) -> None:
    """The C ABI takes raw pointers: the working images must be contiguous 2-D
    CUDA tensors of the precision's type (float32 / float64) whose block grid is
    the plan's, the masks uint8 of the same shape -- anything else would be
    read as the wrong type or past the end."""
    import torch

    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    if len(images_dev) != len(plans) or len(masks_dev) != len(plans):
        raise ValueError("one image and one mask per plan")
    want = torch.float32 if precision == "fp32" else torch.float64
    for i, (t, m, P) in enumerate(zip(images_dev, masks_dev, plans)):
        if t.dtype != want:
            raise ValueError(f"image {i} is {t.dtype}, precision {precision!r} needs {want}")
        if not (t.is_cuda and t.is_contiguous() and m.is_cuda and m.is_contiguous()):
            raise ValueError(f"image/mask {i} must be contiguous CUDA tensors")
        if t.dim() != 2 or m.dtype != torch.uint8 or tuple(m.shape) != tuple(t.shape):
            raise ValueError(f"image/mask {i} must be 2-D of one shape, the mask uint8")
        H, W = t.shape
        if (-(-H // block_size), -(-W // block_size)) != (P.rows, P.cols):
            raise ValueError(f"image {i} of {H}x{W} does not match the plan's {P.rows}x{P.cols} blocks")


def run_frames_device(plans, images_dev, masks_dev, masks_out_dev, params: FseParams,
                      precision: str, picks_dev=None, stream=None) -> None:
    """Run the level pipeline on device tensors already in HBM (the `value` path)."""
    import torch

    n = len(plans)
    if n == 0:
        return
    check_device_frames(images_dev, masks_dev, plans, precision, params.block_size)
    P0 = plans[0]
    F = params.fft_dims((P0.max_wr, P0.max_wc))
    if params.fft_size is not None and (F[0] < P0.max_wr or F[1] < P0.max_wc):
        raise ValueError(f"fft_size {F} smaller than the largest window {(P0.max_wr, P0.max_wc)}")
    dim = max(P0.max_wr, P0.max_wc, 1)
    decay = DeviceContext.decay(params, dim)
    vp = ctypes.c_void_p * n
    pl = vp(*[p.handle.value for p in plans])
    im = vp(*[t.data_ptr() for t in images_dev])
    mk = vp(*[t.data_ptr() for t in masks_dev])
    mo = vp(*[t.data_ptr() for t in masks_out_dev]) if masks_out_dev is not None else None
    code = _lib.FSE_F64 if precision == "fp64" else _lib.FSE_F32
    pc = params.to_c()
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().fse_conceal_frames(
        n, pl, im, mk, mo, ctypes.byref(pc), code, decay.data_ptr(), dim,
        picks_dev.data_ptr() if picks_dev is not None else None, s))


def plan_and_run(masks_host, images_dev, masks_dev, masks_out_dev, params: FseParams,
                 precision: str, order: str = OPTIMIZED, plan_threads: int = 0,
                 first_chunk: int | None = None) -> list:
    """Plan n frames on host threads and run them on the device, overlapping the
    two: the first chunk (~1/8 of the frames) is planned and its level launches
    queued, then the remaining frames are planned while the GPU works on it.
    Returns the plans (in frame order).  Device work is queued on the current
    stream; nothing is synchronised."""
    n = len(masks_host)
    if n == 0:
        return []
    # batches of up to 16 frames run as one session: a first chunk of one or two
    # frames is a dependency-bound session of its own (config-4 frames, fp64, one
    # B200: 8 frames 81.6 ms as 1 + 7 vs 70.6 ms as one session, 16 frames 139.2
    # vs 135.1 ms, 32 frames 266.1 vs 263.3 ms -- there the exposed plan of a
    # single call costs more than that; FSE_CHUNK_MIN sets the threshold)
    k0 = n if n < int(os.environ.get("FSE_CHUNK_MIN", "17")) else (first_chunk or max(1, -(-n // 8)))
    plans = build_plans(masks_host[:k0], params, order, plan_threads)
    if n == 1:  # one frame: its levels are the launches, balance them (multi-frame levels merge across frames)
        balance_for_device(plans[0], params, precision)
    else:
        balance_batch(plans, params, precision)
    run_frames_device(plans, images_dev[:k0], masks_dev[:k0],
                      None if masks_out_dev is None else masks_out_dev[:k0], params, precision)
    if k0 < n:
        rest = build_plans(masks_host[k0:], params, order, plan_threads)
        balance_batch(rest, params, precision)
        run_frames_device(rest, images_dev[k0:], masks_dev[k0:],
                          None if masks_out_dev is None else masks_out_dev[k0:], params, precision)
        plans += rest
    return plans


def _report(plan: Plan, order, threads, wall) -> ConcealReport:
    return ConcealReport(order=order, threads=threads, blocks_processed=plan.n_processed,
                         wall_time=wall, batches=plan.batches(),
                         unconcealed_blocks=plan.unconcealed(), levels=plan.n_levels)


def conceal(image, mask, params: FseParams | None = None, order: str = OPTIMIZED,
            threads: int = 1, precision: str = "fp64", return_picks: bool = False):
    """Conceal every lost block (conceal.py:97-181); see the module docstring."""
    params = _validate(image, mask, params, order, threads, precision)
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("conceal() needs a CUDA device (no CPU fallback)")
    img = np.array(image, dtype=np.float64, copy=True)
    msk = np.array(mask, dtype=np.uint8, copy=True)
    t0 = time.perf_counter()
    plan = build_plan(msk, params, order)
    balance_for_device(plan, params, precision)
    tdt = torch.float64 if precision == "fp64" else torch.float32
    img_d = torch.from_numpy(img).to(device="cuda", dtype=tdt)
    msk_d = torch.from_numpy(msk).cuda()
    out_d = torch.empty_like(msk_d)
    picks_d = None
    if return_picks:
        picks_d = torch.zeros((plan.rows * plan.cols, max(params.iterations, 1), 2),
                              dtype=torch.int32, device="cuda")
    run_frames_device([plan], [img_d], [msk_d], [out_d], params, precision, picks_d)
    out_img = img_d.double().cpu().numpy()
    out_msk = out_d.cpu().numpy()
    wall = time.perf_counter() - t0
    rep = _report(plan, order, threads, wall)
    if return_picks:
        return out_img, out_msk, rep, picks_d[:, : params.iterations].cpu().numpy()
    return out_img, out_msk, rep


_COPY_STREAMS: dict = {}


def _copy_stream():
    """One side stream per device for conceal_batch's overlapped copies."""
    import torch

    dev = torch.cuda.current_device()
    s = _COPY_STREAMS.get(dev)
    if s is None:
        s = _COPY_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return s


def _chunk_bounds(n: int) -> list:
    """Frame chunk boundaries of conceal_batch's staged pipeline: a small first
    chunk (planned while nothing else can run; the rest is planned while it
    computes), the bulk, and (n >= 16) a small last chunk whose compute hides
    the bulk's download.  Measured on config 4 (64 frames, 12 consecutive
    calls): 1/8, 13/16, 1/16 -> 301 ms per call vs 307 ms for 1/8, 7/8; other
    three- and four-chunk splits measured equal or worse.  FSE_CHUNKS="a,b,..."
    (fractions of n) overrides, for experiments."""
    env = os.environ.get("FSE_CHUNKS")
    if env:
        fr = [float(x) for x in env.split(",")]
    elif n >= 16:
        fr = [1 / 8, 13 / 16, 1 / 16]
    elif n >= 12:  # (8 frames: 78.3 ms per call as one chunk vs 80.9 ms as 1 + 7)
        fr = [1 / 8, 7 / 8]
    else:
        fr = [1.0]
    bounds, acc = [0], 0.0
    for f in fr:
        acc += f
        b = min(n, max(bounds[-1] + 1, int(round(acc * n))))
        if b > bounds[-1]:
            bounds.append(b)
    if bounds[-1] < n:
        bounds.append(n)
    return bounds


_BATCH_BUFS: dict = {}
_TRACE = bool(os.environ.get("FSE_E2E_TRACE"))


def _batch_buffers(n, H, W, in_dtype, tdt):
    """(input-dtype image, working image, mask, mask-out) device buffers of one
    batch shape, kept for the next call (the last shape only)."""
    import torch

    key = (torch.cuda.current_device(), n, H, W, in_dtype, tdt)
    if key not in _BATCH_BUFS:
        _BATCH_BUFS.clear()
        img_d = torch.empty((n, H, W), dtype=tdt, device="cuda")
        img_in = img_d if in_dtype == tdt else torch.empty((n, H, W), dtype=in_dtype, device="cuda")
        msk_d = torch.empty((n, H, W), dtype=torch.uint8, device="cuda")
        _BATCH_BUFS[key] = (img_in, img_d, msk_d, torch.empty_like(msk_d))
    return _BATCH_BUFS[key]


def conceal_batch(images, masks, params: FseParams | None = None, order: str = OPTIMIZED,
                  precision: str = "fp64", plan_threads: int = 0, reports: bool = True,
                  out_images=None, out_masks=None):
    """Frame-parallel concealment of equally sized frames: one plan per frame
    (C++ threads, overlapped with the upload), every dependency level of every
    frame in one launch.

    images: [n, H, W] numpy array or CPU torch tensor (any real dtype; pinned
    torch tensors upload asynchronously), masks: [n, H, W] uint8 likewise.
    Returns (images [n, H, W] numpy in the compute dtype — float64 for "fp64",
    float32 for "fp32" —, masks [n, H, W] uint8, reports or None).
    out_images / out_masks: optional preallocated (pinned) CPU tensors of the
    output shapes and dtypes; results land there (streaming callers reuse them
    instead of pinning fresh buffers every call)."""
    if params is None:
        params = FseParams()
    if order not in ORDERS:
        raise ValueError(f"unknown order {order!r}")
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("conceal_batch() needs a CUDA device (no CPU fallback)")
    imgs = images if isinstance(images, torch.Tensor) else torch.from_numpy(np.asarray(images))
    msks = masks if isinstance(masks, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(masks, dtype=np.uint8)))
    if msks.dtype != torch.uint8:
        raise ValueError("masks must be uint8")
    if tuple(imgs.shape) != tuple(msks.shape) or imgs.dim() != 3:
        raise ValueError("images and masks must both be [n, H, W]")
    t0 = time.perf_counter()
    tdt = torch.float64 if precision == "fp64" else torch.float32
    n, H, W = imgs.shape
    out_img = out_images if out_images is not None else torch.empty((n, H, W), dtype=tdt, pin_memory=True)
    out_msk = out_masks if out_masks is not None else torch.empty((n, H, W), dtype=torch.uint8,
                                                                   pin_memory=True)
    if tuple(out_img.shape) != (n, H, W) or out_img.dtype != tdt:
        raise ValueError("out_images has the wrong shape or dtype")
    if tuple(out_msk.shape) != (n, H, W) or out_msk.dtype != torch.uint8:
        raise ValueError("out_masks has the wrong shape or dtype")
    # Staged pipeline (frames are independent):
    #   main stream: upload chunk 1 -> its levels -> [rest uploaded] -> rest's levels -> download rest
    #   copy stream: upload rest (during chunk 1's levels) -> download chunk 1 (during the rest's)
    # The first chunk (~1/8) is planned while its upload runs, the rest while chunk 1 computes.
    main = torch.cuda.current_stream()
    copy = _copy_stream()
    # device buffers persist across calls of one shape (no allocator traffic,
    # which would serialise the two streams); every call ends synchronised
    img_in, img_d, msk_d, out_d = _batch_buffers(n, H, W, imgs.dtype, tdt)
    mh = msks.numpy()
    bounds = _chunk_bounds(n)

    def upload(lo, hi):
        if img_in is img_d:
            img_d[lo:hi].copy_(imgs[lo:hi], non_blocking=True)
        else:
            img_in[lo:hi].copy_(imgs[lo:hi], non_blocking=True)
            img_d[lo:hi].copy_(img_in[lo:hi])
        msk_d[lo:hi].copy_(msks[lo:hi], non_blocking=True)

    def download(lo, hi):
        out_img[lo:hi].copy_(img_d[lo:hi], non_blocking=True)
        out_msk[lo:hi].copy_(out_d[lo:hi], non_blocking=True)

    trace = [("start", time.perf_counter())] if _TRACE else None
    dev_ev = [] if _TRACE else None  # (label, event on the main stream)

    def mark(what):
        if trace is not None:
            trace.append((what, time.perf_counter()))
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(main)
            dev_ev.append((what, ev))

    # chunk 0 is uploaded on the main stream; the rest on the copy stream while
    # chunk 0 computes.  Each chunk is planned while the previous one computes;
    # every chunk but the last is downloaded on the copy stream while the next
    # one computes.
    lo0, hi0 = bounds[0], bounds[1]
    upload(lo0, hi0)
    up = None
    if len(bounds) > 2:
        with torch.cuda.stream(copy):
            upload(hi0, n)
            up = copy.record_event()
    mark("upload")
    plans = []
    for c in range(len(bounds) - 1):
        lo, hi = bounds[c], bounds[c + 1]
        pl = build_plans(list(mh[lo:hi]), params, order, plan_threads)
        if n == 1:
            balance_for_device(pl[0], params, precision)
        else:
            balance_batch(pl, params, precision)
        mark(f"plan{c}")
        if c == 1:
            main.wait_event(up)
        run_frames_device(pl, list(img_d[lo:hi]), list(msk_d[lo:hi]), list(out_d[lo:hi]), params, precision)
        mark(f"run{c}")
        plans += pl
        if hi < n:
            done = main.record_event()
            with torch.cuda.stream(copy):
                copy.wait_event(done)
                download(lo, hi)
        else:
            download(lo, hi)
    main.wait_stream(copy)
    mark("download")
    main.synchronize()
    mark("sync")
    if trace is not None:
        print("conceal_batch: " + "  ".join(f"{w} {1e3 * (t - trace[i][1]):.1f}"
                                            for i, (w, t) in enumerate(trace[1:])), flush=True)
        # device time between the marks (main stream): what the GPU spent on
        # each stage, as opposed to the host's enqueue time above
        print("  device: " + "  ".join(f"{w} {dev_ev[i][1].elapsed_time(e):.1f}"
                                       for i, (w, e) in enumerate(dev_ev[1:])), flush=True)
    wall = time.perf_counter() - t0
    reps = [_report(p, order, 1, wall) for p in plans] if reports else None
    return out_img.numpy(), out_msk.numpy(), reps


def quantize_psnr_device(images_dev, truth_dev=None, masks_dev=None, quantize: bool = True):
    """Output epilogue on device frames [n, H, W] (fp32/fp64): uint8 frames with
    save_pgm rounding (image.py:79-88) and, given the uint8 originals and the
    masks, the per-frame PSNR over non-KNOWN samples (evalkit.psnr,
    evalkit.py:67-81; +inf when equal, ValueError on an empty region).
    Returns (u8 tensor or None, list of PSNR dB or None)."""
    import torch

    x = images_dev
    if x.dim() == 2:
        x = x[None]
    n = x.shape[0]
    npix = x.shape[1] * x.shape[2]
    code = _lib.FSE_F64 if x.dtype == torch.float64 else _lib.FSE_F32
    out = torch.empty(x.shape, dtype=torch.uint8, device=x.device) if quantize else None
    sums = None
    if truth_dev is not None:
        if masks_dev is None:
            raise ValueError("psnr needs the masks")
        sums = torch.empty((n, 2), dtype=torch.float64, device=x.device)
    s = torch.cuda.current_stream().cuda_stream
    t = truth_dev.reshape(x.shape) if truth_dev is not None else None
    m = masks_dev.reshape(x.shape) if masks_dev is not None else None
    _lib.check(_lib.lib().fse_quantize_psnr(
        n, npix, x.contiguous().data_ptr(), code, t.data_ptr() if t is not None else None,
        m.data_ptr() if m is not None else None, out.data_ptr() if out is not None else None,
        sums.data_ptr() if sums is not None else None, s))
    psnrs = None
    if sums is not None:
        psnrs = []
        for se, cnt in sums.cpu().tolist():
            if cnt == 0:
                raise ValueError("mask selects no samples to compare")
            mse = se / cnt
            psnrs.append(float("inf") if mse == 0.0 else 10.0 * np.log10(255.0 ** 2 / mse))
    return out, psnrs
