"""ctypes binding of libfse_b200.so (the C ABI declared in include/fse_b200.h).

The product has no CPU fallback: if the library is missing this module raises
on first use, naming the build command.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSE_LIB") or os.path.join(_HERE, "libfse_b200.so")

FSE_OK, FSE_EINVAL, FSE_ENOMEM, FSE_ECUDA, FSE_ENOTSUP = 0, -22, -12, -5, -95
FSE_F64, FSE_F32 = 0, 1
FSE_ORDER_OPTIMIZED, FSE_ORDER_LINESCAN = 0, 1
FSE_IPC_HANDLE_BYTES = 72

EXPORTS = (
    "fse_last_error", "fse_version", "fse_run_windows", "fse_plan_build", "fse_plan_build_threads", "fse_plan_build_many",
    "fse_plan_free", "fse_plan_sizes", "fse_plan_batches", "fse_plan_levels", "fse_plan_ranks",
    "fse_plan_rebalance",
    "fse_plan_unconcealed", "fse_plan_export_size", "fse_plan_export", "fse_plan_import", "fse_init_counts", "fse_schedule_all", "fse_conceal_frames",
    "fse_launch_count", "fse_timing_enable", "fse_timing_read", "fse_fma_probe",
    "fse_set_guard", "fse_guard_redo_count", "fse_set_dataflow", "fse_set_groups", "fse_set_track_below",
    "fse_set_wcache", "fse_wcache_stats",
    "fse_shard_open", "fse_shard_levels", "fse_shard_run", "fse_shard_close",
    "fse_ipc_handle", "fse_ipc_open", "fse_ipc_close", "fse_flags_alloc", "fse_flags_free",
    "fse_shard_set_peers", "fse_quantize_psnr",
)


class FseParamsC(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32), ("block_size", ctypes.c_int32), ("iterations", ctypes.c_int32),
        ("fft1", ctypes.c_int32), ("fft2", ctypes.c_int32),
        ("rho", ctypes.c_double), ("delta", ctypes.c_double), ("gamma", ctypes.c_double),
    ]


class FseError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libfse_b200 error {code}: {msg}")
        self.code = code


class FseUnsupported(FseError):
    pass


_LIB = None

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_pi32 = ctypes.POINTER(ctypes.c_int32)


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -m paper_2207_00233_b200.build` "
                "(there is no CPU fallback)"
            )
        # one process per GPU (torchrun): the host planner's threads
        # (fse_plan_build, automatic count) share the node's CPUs among the
        # local ranks instead of each rank taking all of them
        lws = int(os.environ.get("LOCAL_WORLD_SIZE", "1") or 1)
        if lws > 1 and "FSE_PLAN_THREADS" not in os.environ:
            os.environ["FSE_PLAN_THREADS"] = str(max(1, (3 * len(os.sched_getaffinity(0))) // (4 * lws)))
        L = ctypes.CDLL(LIB_PATH)
        L.fse_last_error.restype = ctypes.c_char_p
        L.fse_version.argtypes = [_pi32, _i32]
        L.fse_run_windows.argtypes = [_i32, _i32, _i32, _i32, _i32, _vp, _vp, _i32, ctypes.c_double,
                                      _i32, _vp, _vp, _vp, _vp, _vp]
        L.fse_plan_build.argtypes = [_vp, _i32, _i32, ctypes.POINTER(FseParamsC), _i32,
                                     ctypes.POINTER(_vp)]
        L.fse_plan_build_threads.argtypes = [_vp, _i32, _i32, ctypes.POINTER(FseParamsC), _i32, _i32,
                                             ctypes.POINTER(_vp)]
        L.fse_plan_build_many.argtypes = [_i32, ctypes.POINTER(_vp), _i32, _i32,
                                          ctypes.POINTER(FseParamsC), _i32, _i32, ctypes.POINTER(_vp)]
        L.fse_plan_free.argtypes = [_vp]
        L.fse_plan_free.restype = None
        for name in ("fse_plan_batches", "fse_plan_levels"):
            getattr(L, name).argtypes = [_vp, _pi32, _pi32]
        for name in ("fse_plan_sizes", "fse_plan_ranks", "fse_plan_unconcealed"):
            getattr(L, name).argtypes = [_vp, _pi32]
        L.fse_plan_rebalance.argtypes = [_vp, _i32, _i32, _pi32]
        L.fse_plan_export_size.argtypes = [_vp]
        L.fse_plan_export_size.restype = ctypes.c_int64
        L.fse_plan_export.argtypes = [_vp, _vp, ctypes.c_int64]
        L.fse_plan_import.argtypes = [_vp, ctypes.c_int64, ctypes.POINTER(_vp)]
        L.fse_init_counts.argtypes = [_vp, _i32, _i32, _pi32]
        L.fse_schedule_all.argtypes = [_pi32, _i32, _i32, _pi32, _pi32, _pi32]
        L.fse_conceal_frames.argtypes = [_i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                         ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                         ctypes.POINTER(FseParamsC), _i32, _vp, _i32, _vp, _vp]
        L.fse_timing_enable.argtypes = [_i32]
        L.fse_timing_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int64)]
        L.fse_fma_probe.argtypes = [_i32, _i32, _i32, _i32, _vp, _vp]
        L.fse_set_guard.argtypes = [ctypes.c_double, ctypes.c_double]
        L.fse_guard_redo_count.argtypes = [_i32]
        L.fse_set_dataflow.argtypes = [_i32]
        L.fse_set_groups.argtypes = [_i32]
        L.fse_set_track_below.argtypes = [_i32]
        L.fse_set_wcache.argtypes = [_i32]
        _pi64 = ctypes.POINTER(ctypes.c_int64)
        L.fse_wcache_stats.argtypes = [_pi64, _pi64, _pi64, _i32]
        L.fse_shard_open.argtypes = [_vp, _i32, _i32, _vp, _vp, _vp, ctypes.POINTER(FseParamsC), _i32,
                                     _vp, _i32, _vp, ctypes.POINTER(_vp)]
        L.fse_shard_levels.argtypes = [_vp, _pi32, _pi32]
        L.fse_shard_run.argtypes = [_vp, _i32, _i32, _vp]
        L.fse_shard_close.argtypes = [_vp, _vp]
        L.fse_ipc_handle.argtypes = [_vp, _vp]
        L.fse_ipc_open.argtypes = [_vp, ctypes.POINTER(_vp)]
        L.fse_ipc_close.argtypes = [_vp]
        L.fse_flags_alloc.argtypes = [ctypes.POINTER(_vp)]
        L.fse_flags_free.argtypes = [_vp]
        L.fse_shard_set_peers.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_uint32]
        L.fse_quantize_psnr.argtypes = [_i32, ctypes.c_int64, _vp, _i32, _vp, _vp, _vp, _vp, _vp]
        L.fse_guard_redo_count.restype = ctypes.c_int64
        L.fse_launch_count.argtypes = [_i32]
        L.fse_launch_count.restype = ctypes.c_int64
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    if rc != FSE_OK:
        msg = lib().fse_last_error().decode(errors="replace")
        if rc == FSE_EINVAL:
            raise ValueError(msg)
        if rc == FSE_ENOTSUP:
            raise FseUnsupported(rc, msg)
        raise FseError(rc, msg)


def ptr32(a):
    return a.ctypes.data_as(_pi32)


def exports_present() -> list[str]:
    """Names of include/fse_b200.h entry points the loaded library exports."""
    L = lib()
    return [n for n in EXPORTS if hasattr(L, n)]
