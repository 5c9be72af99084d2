"""Weight-spectrum cache of a device session (csrc/fse_wcache.cu): windows
that share their shape and class map load one W = fft2(w)
(fsefill/_kernel.pyx:148, weights fse.py:105-119) instead of computing it.
The cache must never change a bit of the result, whatever its capacity, and
the cached path must reproduce the reference's golden outputs."""

import ctypes
import os

import numpy as np
import pytest

from helpers import conceal_case
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2207_00233_b200")
from paper_2207_00233_b200 import _lib, synth  # noqa: E402


class _Env:
    """FSE_WCACHE_* are read at every session open."""

    def __init__(self, **kv):
        self.kv = {k: str(v) for k, v in kv.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _stats(fn):
    """Run fn with the library's timing on; (result, windows, hits, planes)."""
    L = _lib.lib()
    L.fse_timing_read(None, None, None)
    L.fse_wcache_stats(None, None, None, 1)
    L.fse_timing_enable(1)
    try:
        out = fn()
    finally:
        L.fse_timing_enable(0)
    L.fse_timing_read(None, None, None)
    w, h, p = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    assert L.fse_wcache_stats(ctypes.byref(w), ctypes.byref(h), ctypes.byref(p), 1) == 0
    return out, w.value, h.value, p.value


FORCE = dict(FSE_WCACHE_ENTRIES=1, FSE_WCACHE_MIN_F=32, FSE_WCACHE_WIDTH=0)


@pytest.mark.parametrize("prec,B,F,crop", [
    ("fp64", 4, 64, (160, 224)), ("fp32", 4, 64, (160, 224)),
    ("fp64", 4, 64, (150, 213)),  # ragged: clipped windows of many shapes
    ("fp64", 8, 128, (128, 192)), ("fp32", 8, 128, (128, 192)),
    ("fp64", 2, 32, (96, 128)), ("fp32", 2, 32, (96, 128)),
])
def test_cache_never_changes_a_bit(prec, B, F, crop):
    img, mask = synth.config_scene(5 if B != 4 else 4)
    img, mask = img[:crop[0], :crop[1]].copy(), mask[:crop[0], :crop[1]].copy()
    p = P.FseParams(d=14, iterations=40, block_size=B, fft_size=F)
    L = _lib.lib()
    try:
        assert L.fse_set_wcache(0) == 0
        off, moff, rep = P.conceal(img, mask, p, precision=prec)
        assert L.fse_set_wcache(1) == 0
        results = {}
        for name, env in [("shared", {}), ("every map", dict(FSE_WCACHE_MIN=1)),
                          ("3 planes", dict(FSE_WCACHE_PLANES=3)), ("1 plane", dict(FSE_WCACHE_PLANES=1, FSE_WCACHE_MIN=1))]:
            with _Env(**FORCE, **env):
                (o, m, _), windows, hits, planes = _stats(lambda: P.conceal(img, mask, p, precision=prec))
            assert o.tobytes() == off.tobytes(), name
            np.testing.assert_array_equal(m, moff)
            results[name] = (windows, hits, planes)
        n = rep.blocks_processed
        assert results["shared"][0] == n and 0 < results["shared"][1] <= n
        # every map gets a plane: every window is served from the cache
        assert results["every map"][1] == n
        assert results["3 planes"][1] <= results["shared"][1]
        assert results["1 plane"][1] >= 1
    finally:
        L.fse_set_wcache(1)


@pytest.mark.parametrize("i", [0, 2, 4, 8])
def test_cached_path_matches_reference_golden(golden, i):
    """The golden cases with every window served from the cache (min count 1)."""
    c = conceal_case(golden("conceal_cases.npz"), i)
    if c["fft"] is None or c["fft"][0] != c["fft"][1] or c["fft"][0] not in (32, 64, 128):
        pytest.skip("not a fast-path DFT size")
    p = P.FseParams(d=c["d"], rho=c["rho"], delta=c["delta"], gamma=c["gamma"],
                    iterations=c["iterations"], block_size=c["block_size"], fft_size=c["fft"])
    with _Env(**FORCE, FSE_WCACHE_MIN=1):
        (img, msk, rep, picks), windows, hits, _ = _stats(
            lambda: P.conceal(c["image"], c["mask"], p, c["order"], precision="fp64", return_picks=True))
    assert hits == windows == rep.blocks_processed
    np.testing.assert_array_equal(msk, c["out_mask"])
    assert rep.batches == c["batches"]
    assert np.max(np.abs(img - c["out_image"])) <= 1e-6
    for b, want in zip(c["pick_blocks"].tolist(), c["picks"]):
        assert O.canonical_picks(picks[b], c["fft"]) == [tuple(x) for x in want.tolist()], b


def test_cache_in_batches_and_default_threshold():
    """conceal_batch over several frames shares planes across frames; small
    sessions (below the FSE_WCACHE_ENTRIES / FSE_WCACHE_ENTRIES_ALL window counts)
    leave the cache off."""
    sc = [synth.config_scene(4, f) for f in range(3)]
    imgs = np.stack([s[0][:160, :224] for s in sc])
    msks = np.stack([s[1][:160, :224] for s in sc])
    p = P.FseParams(d=14, iterations=30, block_size=4, fft_size=64)
    L = _lib.lib()
    try:
        L.fse_set_wcache(0)
        off, moff, _ = P.conceal_batch(imgs, msks, p, precision="fp64", reports=False)
        L.fse_set_wcache(1)
        with _Env(**FORCE):
            (on, mon, _), windows, hits, planes = _stats(
                lambda: P.conceal_batch(imgs, msks, p, precision="fp64", reports=False))
        assert on.tobytes() == off.tobytes() and mon.tobytes() == moff.tobytes()
        assert hits > 0 and planes > 0
        (dflt, _, _), windows, hits, planes = _stats(
            lambda: P.conceal_batch(imgs, msks, p, precision="fp64", reports=False))
        assert dflt.tobytes() == off.tobytes()
        assert windows == 0 or windows >= 1024  # default thresholds (FSE_WCACHE_ENTRIES / _ENTRIES_ALL)
    finally:
        L.fse_set_wcache(1)
