"""FSE throughput benchmark (BASELINE.json metric: lost blocks/s and lost
Mpixel/s, plus the fraction of the FP32 CUDA-core roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config 4] [--precision fp64] [--frames 64] [--defaults]

Workload (N=1 and every N): BASELINE config 4 — 64 independent 1920x1080
synthetic luma frames (per-frame seeds), 20% mixed isolated+burst 16x16
losses, FSE 4x4 / d=14 / FFT 64x64 / 100 iterations, rho=0.8, gamma=0.5,
delta=0.2, optimized order, fp64 (the parity path: identical picks to the
reference, samples within 1e-6; --precision fp32 is the non-parity fast mode,
also measured as a secondary record).  Frame-parallel: rank r of N owns a
contiguous 64/N frame range (no data-path collective; scaling "strong": the
64-frame job is fixed).  One step = the whole job once:
    uint8->float working copy -> host C++ plans of the rank's frames, the first
    1/8 of them planned and launched before the rest is planned (overlapping the
    GPU) -> every dependency level of a chunk's frames as one sm_100a launch ->
    mask pass.
value = lost FSE blocks of all ranks / max-over-ranks device time of K steps,
inputs resident in HBM.  e2e = the same through the public conceal_batch()
with pinned host frames in and results out (H2D/D2H inside the region).

--impl reference: the reference's own compiled FSE kernel (oracle/_ref, i.e.
fsefill._kernel.run_fse) driven by the oracle's restatement of conceal()
(optimized order), frame-parallel over all host cores (one process per core,
each a different frame), each step a bounded sample of the same workload.
Rank 0 only; other ranks exit 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

B, D, F, RHO, DELTA, GAMMA = 4, 14, 64, 0.8, 0.2, 0.5


def counted_flops_per_block(iters: int, f1: int, f2: int) -> float:
    """17 * I * F1 * (F2/2 + 1) algorithmic FLOPs per block."""
    return 17.0 * iters * f1 * (f2 // 2 + 1)


PARITY = {
    "fp64": "parity path: every block's canonical pick sequence identical to the reference's and every "
            "sample within 1e-6 (tests/test_gpu_conceal.py: 11 golden cases, full configs 1-4 and a 4K crop)",
    "fp32": "NOT parity-green: fp32 fast mode; near-tie pick switches move some samples by more than 0.5 "
            "(DESIGN.md §5) -- reported for reference only",
}


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--block", type=int, default=4, choices=[2, 4, 8],
                    help="config 5 block size (FFT 32 / 64 / 128)")
    ap.add_argument("--precision", default="fp64", choices=["fp32", "fp64"],
                    help="fp64 = the parity path (identical picks, 1e-6; the headline); fp32 = the "
                         "non-parity fast mode (DESIGN.md §5)")
    ap.add_argument("--defaults", action="store_true",
                    help="the reference's default parameters (FseParams(): B=16, d=16, I=200, DFT = window "
                         "size) -- the drop-in call conceal(image, mask) -- on the config's frames")
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--guard", default=None,
                    help="fp32 near-tie guard 'tau0,tau1' or 'off' (default: library default)")
    ap.add_argument("--plan-on", default="rank0", choices=["rank0", "all"],
                    help="config 5 at N>1: plan the frame on rank 0 and broadcast it (default), or on every rank")
    ap.add_argument("--halo", default="p2p", choices=["p2p", "collective"],
                    help="config 5 at N>1: fused halo stores over peer memory (default) or per-level "
                         "send/recv over torch.distributed")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-second", action="store_true", help="skip the other precision's measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-blocks", type=int, default=5200,
                    help="cpu_baseline sample: lossy blocks of frame 0 (about 10 s on one core of the GPU box)")
    return ap.parse_args()


def iterations_for(config):
    return 200 if config == 3 else 100


def frame_ids(config, frames, rank, world):
    n = frames if config == 4 else 1
    lo, hi = rank * n // world, (rank + 1) * n // world
    return list(range(lo, hi))


def make_scenes(config, ids, threads=None):
    from concurrent.futures import ThreadPoolExecutor

    from paper_2207_00233_b200 import synth

    with ThreadPoolExecutor(max_workers=threads or min(16, os.cpu_count() or 1)) as ex:
        return list(ex.map(lambda f: synth.config_scene(config, f), ids))


def workload_name(config, frames, precision, defaults=False):
    if defaults:
        return (f"config{config}: {frames if config == 4 else 1} x 1920x1080 synthetic luma, reference DEFAULT "
                f"parameters FseParams() (B=16, d=16, I=200, rho=0.8, delta=0.2, gamma=0.5, DFT = window "
                f"size 48x48 / clipped), optimized order, {precision}")
    if config == 4:
        return (f"config4: {frames} x 1920x1080 synthetic luma frames, 20% mixed 16x16 losses, "
                f"FSE 4x4 / d=14 / FFT 64x64 / 100 it, optimized order, {precision}, frame-parallel")
    return (f"config3: 1920x1080 synthetic luma, 30% isolated 16x16 losses, FSE 4x4 / d=14 / "
            f"FFT 64x64 / 200 it, optimized order, {precision}")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        # nvidia-smi -i takes a physical index or a UUID; the UUID survives any
        # CUDA_VISIBLE_DEVICES remapping
        self.index = index
        try:
            import torch

            u = str(torch.cuda.get_device_properties(index % max(1, torch.cuda.device_count())).uuid)
            self.index = u if u.startswith("GPU-") else f"GPU-{u}"
        except Exception:
            pass
        self.rows = []
        self._p = None
        self._t = None

    def _run(self):
        # ONE nvidia-smi process in loop mode (-lms 200), started before the timed
        # region and killed after it, as the profiling recipe does: a process per
        # sample costs ~0.3 s of host CPU and a driver lock each, which showed up as
        # host stalls inside the timed steps (step 588-779 ms against 519 ms of kernels)
        for line in self._p.stdout:
            row = [x.strip() for x in line.strip().split(",")]
            if len(row) == 6:
                self.rows.append(row)
                self._first.set()

    def __enter__(self):
        self._first = threading.Event()
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._p = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._first.wait(3.0)  # the process is up and sampling before the timed region starts
        self._start = len(self.rows)  # samples taken before the region are not "under load"
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        self._p.terminate()
        try:
            self._p.wait(timeout=3)
        except Exception:
            self._p.kill()
        self._t.join(timeout=3)

    def summary(self):
        # a region shorter than the sampling period keeps the sample taken just before it
        self.rows = self.rows[getattr(self, "_start", 0):] or self.rows[-1:]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ reference arm

def oracle_params(O, iters, defaults):
    """The oracle's Params for the bench workload (or the reference defaults)."""
    if defaults:
        return O.Params()  # fse.py:55-86 defaults, DFT = window size
    return O.Params(d=D, rho=RHO, delta=DELTA, gamma=GAMMA, iterations=iters, block_size=B, fft_size=(F, F))


def _ref_worker(job):
    config, frame, iters, limit, defaults = job
    from oracle import oracle as O
    from paper_2207_00233_b200 import synth

    img, mask = synth.config_scene(config, frame)
    p = oracle_params(O, iters, defaults)
    kernel = "ref" if O.ref_kernel() is not None else "c"
    _, _, rep = O.conceal(img, mask, p, "optimized", kernel=kernel, block_limit=limit)
    return rep.blocks_processed, sample_seconds(rep), kernel


def sample_seconds(rep):
    """CPU time the reference would spend on the sampled blocks: their fits plus
    the frame's scheduling cost amortised over its lossy blocks (the reference's
    conceal() schedules the whole frame up front, conceal.py:145)."""
    fit = rep.wall_time - rep.sched_time
    return fit + rep.sched_time * rep.blocks_processed / max(1, rep.n_lossy)


def cpu_reference(config, iters, cores, blocks_per_core, frames, defaults=False):
    """Frame-parallel CPU run of the reference kernel: one process per core, each
    concealing the first `blocks_per_core` blocks of a different frame."""
    import multiprocessing as mp

    jobs = [(config, f % (frames if config == 4 else 1), iters, blocks_per_core, defaults) for f in range(cores)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        res = pool.map(_ref_worker, jobs)
    # workers run concurrently; the step lasts as long as the slowest one
    # (scene generation and process start-up are excluded)
    blocks = sum(r[0] for r in res)
    return blocks, max(r[1] for r in res), res[0][2]


def host_cores():
    """(usable logical CPUs of this process, physical cores of the host)."""
    cores = os.cpu_count() or 1
    physical = None
    try:
        import psutil

        cores = len(psutil.Process().cpu_affinity()) or cores
        physical = psutil.cpu_count(logical=False)
    except Exception:
        pass
    return cores, physical


def run_reference(a, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O

    iters = iterations_for(a.config)
    cores, physical = host_cores()
    per = max(20, 160 // max(1, iters // 100))  # ~0.75 s of CPU per core per step
    if a.defaults:
        per = 40  # 48x48 windows at 200 iterations: ~4 ms each
    kernel = "ref" if O.ref_kernel() is not None else "c"
    for _ in range(a.warmup):
        cpu_reference(a.config, iters, cores, per // 4, a.frames, a.defaults)
    tot_b, tot_t = 0, 0.0
    lost_px_per_block = (16 if a.defaults else B) ** 2
    for _ in range(a.steps):
        b, t, kernel = cpu_reference(a.config, iters, cores, per, a.frames, a.defaults)
        tot_b += b
        tot_t += t
    value = tot_b / tot_t
    sample = (f"{cores} processes x first {per} lossy blocks (optimized order) of distinct frames "
              f"per step, frame schedule amortised pro rata; "
              f"kernel={'oracle/_ref (reference _kernel.pyx compiled here)' if kernel == 'ref' else 'oracle C port'}")
    line = {
        "impl": "reference", "metric": "lost_blocks_per_s", "value": value, "unit": "blocks/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1000.0 * tot_t / a.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE generators)",
        "config": {"workload": workload_name(a.config, a.frames, "fp64", a.defaults), "sample": sample},
        "lost_mpixel_per_s": value * lost_px_per_block / 1e6,
        "cpu_baseline": {"value": value, "unit": "blocks/s", "cores": cores, "physical_cores": physical,
                         "cores_note": "cores = processes run (one per usable logical CPU); physical_cores "
                                       "= psutil.cpu_count(logical=False) on this host",
                         "kind": "reference" if kernel == "ref" else "port", "sample": sample},
        "e2e": {"value": value, "unit": "blocks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm

def _allreduce(torch, dist, values, op):
    """all_reduce of a few floats on the backend's device (CPU for gloo)."""
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(values, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return t.cpu().tolist()


def measure_peaks(torch, lib):
    """Arithmetic throughput of this GPU (roofline denominators), CUDA events:
    FFMA, FFMA2 (packed f32x2, what the fp32 kernel issues) and DFMA."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    scratch = torch.zeros(1, device="cuda")
    s = torch.cuda.current_stream()
    blocks, threads, iters = sms * 8, 256, 4096
    out = {}
    for kind, name, fpt in ((0, "ffma", 16.0), (1, "ffma2", 32.0), (2, "dfma", 16.0)):
        for _ in range(2):
            lib.fse_fma_probe(kind, blocks, threads, iters, scratch.data_ptr(), s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            lib.fse_fma_probe(kind, blocks, threads, iters, scratch.data_ptr(), s.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[name] = fpt * iters * blocks * threads / (ms * 1e-3) / 1e12
    return out, sms


def run_b200(a, rank, world, local_rank):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2207_00233_b200 as P
    from paper_2207_00233_b200 import _lib

    torch.cuda.set_device(local_rank % max(1, torch.cuda.device_count()))
    lib = _lib.lib()
    if a.guard is not None:
        t0_, t1_ = (-1.0, 0.0) if a.guard == "off" else (float(x) for x in a.guard.split(","))
        lib.fse_set_guard(t0_, t1_)
    iters = iterations_for(a.config)
    params = P.FseParams(d=D, rho=RHO, delta=DELTA, gamma=GAMMA, iterations=iters, block_size=B,
                         fft_size=F)
    if a.defaults:
        params = P.FseParams()  # reference defaults (fse.py:55-86), DFT = window size
        iters = params.iterations
    ids = frame_ids(a.config, a.frames, rank, world)
    scenes = make_scenes(a.config, ids)
    imgs_h = torch.from_numpy(np.stack([s[0] for s in scenes])).pin_memory()
    msks_h = torch.from_numpy(np.stack([s[1] for s in scenes])).pin_memory()
    n, H, W = imgs_h.shape
    imgs_d = imgs_h.cuda()
    msks_d = msks_h.cuda()
    mout = torch.empty_like(msks_d)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    masks_np = list(msks_h.numpy())
    # share the host cores between the ranks of this node (the C++ planner
    # otherwise starts hardware_concurrency threads in every rank)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    plan_threads = max(1, (os.cpu_count() or 1) // max(1, local_world)) if world > 1 else 0

    # work accounting from one plan set
    plans = P.build_plans(masks_np, params, "optimized", plan_threads)
    blocks_rank = sum(p.n_processed for p in plans)
    # counted FLOPs of this rank's blocks: 17 I F1 (F2/2 + 1) each, F = the
    # FFT size or (fft_size=None) the block's own window shape
    if params.fft_size is None:
        flop_rank = 0.0
        for pl in plans:
            blk = np.asarray([b for lv in pl.levels() for b in lv], dtype=np.int64)
            r, c = blk // pl.cols, blk % pl.cols
            Bq, dq = params.block_size, params.d
            Mw = np.minimum(H, np.minimum(r * Bq + Bq, H) + dq) - np.maximum(0, r * Bq - dq)
            Nw = np.minimum(W, np.minimum(c * Bq + Bq, W) + dq) - np.maximum(0, c * Bq - dq)
            flop_rank += float(np.sum(17.0 * iters * Mw * (Nw // 2 + 1)))
    else:
        flop_rank = blocks_rank * counted_flops_per_block(iters, F, F)
    lost_px_rank = int((msks_h == 1).sum())
    levels = max(p.n_levels for p in plans)
    del plans

    def timed(fn, k):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        keep = None
        for _ in range(k):
            keep = fn()
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        del keep
        if world > 1:
            ms = _allreduce(torch, dist, [ms], dist.ReduceOp.MAX)[0]
        return ms

    def measure(precision, sample_clocks):
        """Device-resident step: plans + uint8->float working copy + level
        launches + mask pass, K steps after W warm-up steps."""
        tdt = torch.float32 if precision == "fp32" else torch.float64
        work = torch.empty((n, H, W), dtype=tdt, device="cuda")
        plan_ms = []

        def step():
            flush.zero_()
            work.copy_(imgs_d)
            t = time.perf_counter()
            pl = P.plan_and_run(masks_np, list(work), list(msks_d), list(mout), params, precision,
                                "optimized", plan_threads)
            plan_ms.append(1e3 * (time.perf_counter() - t))
            return pl

        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        plan_ms.clear()
        lib.fse_launch_count(1)
        lib.fse_timing_read(None, None, None)
        lib.fse_guard_redo_count(1)
        lib.fse_wcache_stats(None, None, None, 1)
        lib.fse_timing_enable(1)
        clk = ClockSampler(local_rank) if sample_clocks else None
        if clk:
            clk.__enter__()
        ms = timed(step, a.steps)
        if clk:
            clk.__exit__(None, None, None)
        lib.fse_timing_enable(0)
        launches = int(lib.fse_launch_count(1))
        kms, wl, calls = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.fse_timing_read(ctypes.byref(kms), ctypes.byref(wl), ctypes.byref(calls)))
        redo = int(lib.fse_guard_redo_count(1))
        wcw, wch, wcp = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib.fse_wcache_stats(ctypes.byref(wcw), ctypes.byref(wch), ctypes.byref(wcp), 1)
        wcache = {"windows_per_step": wcw.value / a.steps, "hits_per_step": wch.value / a.steps,
                  "planes_per_step": wcp.value / a.steps,
                  "hit_share": (wch.value / wcw.value) if wcw.value else 0.0}
        return {"ms": ms, "kernel_ms": kms.value / a.steps, "launches": launches, "wcache": wcache,
                "level_launches": int(wl.value),
                "plan_ms": float(np.mean(plan_ms)) if plan_ms else None,
                "plan_ms_steps": [round(x, 1) for x in plan_ms], "redo": redo / a.steps,
                "clocks": clk.summary() if clk else None}

    head = measure(a.precision, True)
    other_prec = "fp64" if a.precision == "fp32" else "fp32"
    other = None if a.no_second else measure(other_prec, False)

    blocks_all, lost_px_all = float(blocks_rank), float(lost_px_rank)
    if world > 1:
        blocks_all, lost_px_all = _allreduce(torch, dist, [blocks_rank, lost_px_rank], dist.ReduceOp.SUM)
    value = blocks_all * a.steps / (head["ms"] * 1e-3)

    # roofline of the dominant kernel (the level launches): counted FLOPs per
    # block x blocks of this rank / summed CUDA-event time of the level launches
    peaks, sms = measure_peaks(torch, lib)
    fp32_peak = max(peaks["ffma"], peaks["ffma2"])

    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic_r4.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))

    def roof(m, precision):
        achieved = flop_rank / (m["kernel_ms"] * 1e-3) / 1e12
        pk = fp32_peak if precision == "fp32" else peaks["dfma"]
        tr, detail = None, None
        blocks_per_launch = blocks_rank * a.steps / max(1, m["level_launches"])
        tp = traffic.get(precision) if traffic else None
        if tp:
            # ncu dram bytes per window x the average windows of a timed launch
            tr = tp["dram_bytes_per_block"] * blocks_per_launch
            detail = {"dram_bytes_per_block": tp["dram_bytes_per_block"],
                      "algorithmic_bytes_per_block": tp["algorithmic_bytes_per_block"],
                      "avg_blocks_per_launch": blocks_per_launch,
                      "profiled_launch": {"blocks": tp["launch_blocks"],
                                          "dram_bytes": tp["dram_bytes_per_launch"]},
                      "source": traffic["source"]}
        return {"bound": "fp32" if precision == "fp32" else "fp64", "achieved": achieved, "peak": pk,
                "unit": "TFLOP/s", "frac": achieved / pk, "frac_of_fp32_peak": achieved / fp32_peak,
                "traffic": tr, "traffic_detail": detail,
                "bound_note": "FP32 (FP64) CUDA-core pipe roofline as BASELINE.json asks; the kernel "
                              "is compute/issue bound (>600 FLOP per HBM byte)",
                "kernel": "fse_fast_kernel (one launch per dependency level)",
                "flops_per_block": flop_rank / max(1, blocks_rank),
                "peak_source": (f"measured live on {sms} SMs by fse_fma_probe: FFMA {peaks['ffma']:.1f}, "
                                f"FFMA2 {peaks['ffma2']:.1f}, DFMA {peaks['dfma']:.1f} TFLOP/s")}

    # e2e through the public API with pinned host buffers
    e2e = None
    if not a.no_e2e:
        # streaming use: the caller's pinned result buffers are allocated once
        out_img_h = torch.empty((n, H, W), dtype=torch.float32 if a.precision == "fp32" else torch.float64,
                                pin_memory=True)
        out_msk_h = torch.empty((n, H, W), dtype=torch.uint8, pin_memory=True)

        def e2e_step():
            return P.conceal_batch(imgs_h, msks_h, params, "optimized", a.precision,
                                   plan_threads, reports=False, out_images=out_img_h,
                                   out_masks=out_msk_h)
        for _ in range(max(1, min(2, a.warmup))):
            e2e_step()
        ems = timed(e2e_step, a.steps)
        esz = 4 if a.precision == "fp32" else 8
        e2e = {"value": blocks_all * a.steps / (ems * 1e-3), "unit": "blocks/s",
               "ms_per_step": ems / a.steps,
               "h2d_bytes_per_step": int(imgs_h.numel() * imgs_h.element_size() + msks_h.numel()) * world,
               "d2h_bytes_per_step": int(n * H * W * (esz + 1)) * world}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle import oracle as O

        img0, m0 = scenes[0]
        p0 = oracle_params(O, iters, a.defaults)
        kern = "ref" if O.ref_kernel() is not None else "c"
        _, _, rep = O.conceal(img0, m0, p0, "optimized", kernel=kern,
                              block_limit=a.cpu_blocks // (8 if a.defaults else 1))
        secs = sample_seconds(rep)
        cpu = {"value": rep.blocks_processed / secs, "unit": "blocks/s", "cores": 1,
               "host_physical_cores": host_cores()[1],
               "kind": "reference" if kern == "ref" else "port",
               "sample": f"first {rep.blocks_processed} of {rep.n_lossy} lossy blocks (optimized order) "
                         f"of frame 0: {rep.wall_time - rep.sched_time:.1f} s of fits + "
                         f"{rep.sched_time:.1f} s frame schedule amortised pro rata, 1 thread; kernel="
                         + ("oracle/_ref = reference _kernel.pyx compiled here" if kern == "ref"
                            else "oracle C port")}

    if rank == 0:
        line = {
            "metric": "lost_blocks_per_s", "value": value, "unit": "blocks/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": head["ms"] / a.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if a.precision == "fp32" else "f64",
            "data": "synthetic (seeded BASELINE generators, paper_2207_00233_b200/synth.py)",
            "config": {"workload": workload_name(a.config, a.frames, a.precision, a.defaults),
                       "frames": len(frame_ids(a.config, a.frames, 0, 1)), "H": H, "W": W,
                       "block": params.block_size, "d": params.d, "fft": params.fft_size,
                       "iterations": iters, "rho": params.rho, "delta": params.delta,
                       "gamma": params.gamma, "order": "optimized",
                       "parallelism": f"frame-parallel x{world}",
                       "l2": "256 MiB buffer written every step (> 126 MB L2)"},
            "lost_mpixel_per_s": lost_px_all * a.steps / (head["ms"] * 1e-3) / 1e6,
            "blocks_per_step": blocks_all, "lost_pixels_per_step": lost_px_all,
            "levels_per_step": levels,
            "host_enqueue_ms_per_step": head["plan_ms"], "host_enqueue_ms_steps": head["plan_ms_steps"],
            "kernel_ms_per_step": head["kernel_ms"],
            "fp32_guard_fp64_redo_per_step": head["redo"],
            "weight_spectrum_cache": head["wcache"],
            "parity": PARITY[a.precision],
            "roofline": roof(head, a.precision),
            "gpu_launches": head["launches"],
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": head["clocks"],
        }
        if other is not None:
            line[other_prec] = {
                "value": blocks_all * a.steps / (other["ms"] * 1e-3), "unit": "blocks/s",
                "ms_per_step": other["ms"] / a.steps, "kernel_ms_per_step": other["kernel_ms"],
                "roofline": roof(other, other_prec), "gpu_launches": other["launches"],
                "parity": PARITY[other_prec]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()


def run_small_bench(a, rank, world, local_rank):
    """BASELINE configs 1 and 2: one 512x512 frame, B=4 / d=14 / FFT 64 /
    100 it.  Config 1: fp64, optimized order.  Config 2: optimized vs line-scan
    order in fp32 and fp64 (the PSNR difference and the speed-up BASELINE asks
    for).  Replicas only: every rank runs the same frame (these configs do not
    shard).  A step = host plan + device levels + mask pass on resident inputs."""
    import torch

    import paper_2207_00233_b200 as P
    from paper_2207_00233_b200 import _lib, synth
    from paper_2207_00233_b200.conceal import balance_for_device

    torch.cuda.set_device(local_rank % max(1, torch.cuda.device_count()))
    params = P.FseParams(d=D, rho=RHO, delta=DELTA, gamma=GAMMA, iterations=100, block_size=B, fft_size=F)
    img, mask = synth.config_scene(a.config)
    truth = img.astype(np.float64)
    msk = torch.from_numpy(mask).cuda()
    out = torch.empty_like(msk)
    lib = _lib.lib()

    def run(order, precision):
        tdt = torch.float32 if precision == "fp32" else torch.float64
        src = torch.from_numpy(img).cuda().to(tdt)
        work = torch.empty_like(src)

        def step():
            work.copy_(src)
            plan = P.build_plan(mask, params, order)
            balance_for_device(plan, params, precision)
            P.run_frames_device([plan], [work], [msk], [out], params, precision)
            return plan

        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            plan = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        res = work.double().cpu().numpy()
        region = mask != 0
        mse = float(np.mean((truth[region] - res[region]) ** 2))
        return {"ms": ms, "blocks": plan.n_processed, "levels": plan.n_levels, "batches": plan.n_batches,
                "psnr_db": 10 * np.log10(255.0 ** 2 / mse)}

    lib.fse_launch_count(1)
    combos = [("optimized", "fp64")] if a.config == 1 else [
        ("optimized", "fp32"), ("linescan", "fp32"), ("optimized", "fp64"), ("linescan", "fp64")]
    res = {f"{o}_{p}": run(o, p) for o, p in combos}
    launches = int(lib.fse_launch_count(1))
    head = res["optimized_fp64"]  # the parity path
    if rank == 0:
        line = {
            "metric": "lost_blocks_per_s", "value": head["blocks"] / (head["ms"] * 1e-3), "unit": "blocks/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": head["ms"],
            "higher_is_better": True, "scaling": "replicas", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded BASELINE generators, paper_2207_00233_b200/synth.py)",
            "config": {"workload": f"config{a.config}: 512x512 synthetic, "
                                   + ("10% isolated" if a.config == 1 else "20% horizontal bursts")
                                   + " 16x16 losses, FSE 4x4 / d=14 / FFT 64x64 / 100 it"},
            "lost_mpixel_per_s": float((mask == 1).sum()) / (head["ms"] * 1e-3) / 1e6,
            "runs": res, "gpu_launches": launches,
        }
        if a.config == 2:
            for p in ("fp32", "fp64"):
                o, l = res[f"optimized_{p}"], res[f"linescan_{p}"]
                line[f"{p}_optimized_minus_linescan_psnr_db"] = o["psnr_db"] - l["psnr_db"]
                line[f"{p}_optimized_speedup_over_linescan"] = l["ms"] / o["ms"]
        print(json.dumps(line), flush=True)


def run_strips_bench(a, rank, world, local_rank):
    """BASELINE config 5: one 3840x2160 frame, 50% burst losses, B in {2,4,8}
    (FFT 32/64/128), 100 iterations, --precision (fp64 default), spatially strip-sharded over the
    ranks (paper_2207_00233_b200.strips).  A step = host plan (every rank, same
    global plan) + shard levels with halo exchanges + result gather to rank 0."""
    import torch
    import torch.distributed as dist

    import paper_2207_00233_b200 as P
    from paper_2207_00233_b200 import _lib, strips, synth
    from paper_2207_00233_b200.conceal import balance_for_device

    torch.cuda.set_device(local_rank % max(1, torch.cuda.device_count()))
    Bk = a.block
    Fk = {2: 32, 4: 64, 8: 128}[Bk]
    params = P.FseParams(d=D, rho=RHO, delta=DELTA, gamma=GAMMA, iterations=100, block_size=Bk,
                         fft_size=Fk)
    img, mask = synth.config_scene(5)
    H, W = mask.shape
    src = torch.from_numpy(img).cuda().to(torch.float32 if a.precision == "fp32" else torch.float64)
    msk = torch.from_numpy(mask).cuda()
    work = torch.empty_like(src)
    out = torch.empty_like(msk)
    R = strips.halo_rows(params)
    grp = dist.group.WORLD if world > 1 else None
    stats = {}
    # fused halo exchange: the frame buffer is fixed, so its peer mappings are
    # set up once; each step is a new epoch of the device flags
    # (None on every rank when some rank cannot map its neighbours: the
    # per-level collective exchange then runs instead, and the line says so)
    link = strips.open_peer_link(work, rank, world, dist, grp) if world > 1 and a.halo == "p2p" else None
    hg = strips.host_group(dist, grp) if world > 1 and a.plan_on == "rank0" else None

    def step():
        work.copy_(src)
        t0 = time.perf_counter()
        if hg is not None:  # plan once, broadcast the bytes over a host (gloo) group
            plan = strips.broadcast_plan(mask, params, "optimized", rank, dist, hg, 0, precision=a.precision)
        else:
            plan = P.build_plan(mask, params)
            balance_for_device(plan, params, a.precision)
        processed = (plan.ranks() != np.iinfo(np.int32).max).reshape(plan.rows, plan.cols)
        bands = strips.band_partition(processed.sum(axis=1), world, R)
        stats["plan_ms"] = 1e3 * (time.perf_counter() - t0)
        stats["blocks"] = plan.n_processed
        ex = strips.ShardExecutor(plan, bands[rank], work, msk, out, params, a.precision)
        if link is not None and strips.run_levels_p2p(ex, link, dist, grp):
            stats["halo_msgs"] = 0
            stats["fused"] = True
        else:
            stats["fused"] = False
            stats["halo_msgs"] = strips.run_levels_collective(ex, work, rank, world, bands, R, Bk, H, dist, grp)
        stats["levels"] = ex.n_levels
        ex.close()
        if world > 1:  # gather the bands to rank 0 (gloo: through host buffers)
            lo, hi = bands[rank]
            host = dist.get_backend() == "gloo"
            if rank == 0:
                for r in range(1, world):
                    y0, y1 = bands[r][0] * Bk, min(H, bands[r][1] * Bk)
                    if host:
                        hb = work[y0:y1].cpu()
                        dist.recv(hb, r)
                        work[y0:y1].copy_(hb)
                    else:
                        dist.recv(work[y0:y1], r)
            else:
                rows = work[lo * Bk:min(H, hi * Bk)].contiguous()
                dist.send(rows.cpu() if host else rows, 0)
        return plan

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lib = _lib.lib()
    lib.fse_launch_count(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record()
        for _ in range(a.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        ms = _allreduce(torch, dist, [ms], dist.ReduceOp.MAX)[0]
    launches = int(lib.fse_launch_count(1))
    strips_equal = None
    if world > 1 and rank == 0:
        # the gathered strip-sharded frame against one whole-frame run on this
        # GPU (same kernels; untimed)
        whole = src.clone()
        wout = torch.empty_like(msk)
        P.run_frames_device([P.build_plan(mask, params)], [whole], [msk], [wout], params, a.precision)
        torch.cuda.synchronize()
        strips_equal = bool(torch.equal(whole, work))
    if rank == 0:
        blocks = stats["blocks"]
        flop = counted_flops_per_block(100, Fk, Fk) * blocks
        line = {
            "metric": "lost_blocks_per_s", "value": blocks * a.steps / (ms * 1e-3), "unit": "blocks/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32" if a.precision == "fp32" else "f64",
            "data": "synthetic (seeded BASELINE generators, paper_2207_00233_b200/synth.py)",
            "config": {"workload": f"config5: 3840x2160 synthetic luma, 50% burst 16x16 losses, FSE "
                                   f"{Bk}x{Bk} / d=14 / FFT {Fk}x{Fk} / 100 it, optimized order, {a.precision}, "
                                   f"strip-sharded", "block": Bk, "fft": Fk,
                       "parallelism": f"row bands x{world}, halo exchange: "
                                      + ("fused peer stores + device flags" if link is not None
                                         else "per-level send/recv" if world > 1 else "none")
                                      + (", plan on rank 0 + broadcast" if hg is not None else "")},
            "lost_mpixel_per_s": float((mask == 1).sum()) * a.steps / (ms * 1e-3) / 1e6,
            "blocks_per_step": blocks, "levels_per_step": stats["levels"],
            "host_plan_ms_per_step": stats["plan_ms"], "halo_messages_rank0": stats["halo_msgs"],
            "counted_tflop_per_s": flop * a.steps / (ms * 1e-3) / 1e12,
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        if strips_equal is not None:
            line["strips_equal_whole_frame"] = strips_equal
        print(json.dumps(line), flush=True)
    if link is not None:
        torch.cuda.synchronize()
        dist.barrier()
        link.close()


def main():
    a = args_()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != a.gpus and "RANK" in os.environ:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    import torch
    import torch.distributed as dist

    if world > 1:
        # FSE_BENCH_BACKEND=gloo: functional multi-rank check on a single GPU
        # (ranks share the device; only host-side barriers/reductions, no
        # kernel waits on another rank) — numbers from such a run are not valid
        backend = os.environ.get("FSE_BENCH_BACKEND", "nccl")
        dev = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    try:
        if a.config == 5:
            run_strips_bench(a, rank, world, local_rank)
        elif a.config in (1, 2):
            run_small_bench(a, rank, world, local_rank)
        else:
            run_b200(a, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
