"""Reporting harness (evalkit.py:67-160 restated in paper_2207_00233_b200.evalkit):
PSNR closed forms and the CSV layout on the CPU, the bench sweep on the GPU."""

import io

import numpy as np
import pytest

from paper_2207_00233_b200 import evalkit as E


def test_psnr_closed_forms_and_region():
    base = np.zeros((10, 10))
    mask = np.zeros((10, 10), np.uint8)
    mask[:4, :] = E.LOST
    off = base.copy()
    off[:4, :] += 16.0
    assert E.psnr(base, off, mask) == pytest.approx(10 * np.log10(255 ** 2 / 256))
    worst = base.copy()
    worst[:4, :] += 255.0
    assert E.psnr(base, worst, mask) == pytest.approx(0.0, abs=1e-12)
    assert E.psnr(base, base.copy(), mask) == float("inf")
    # reconstructed (2) counts like lost; known samples never do
    m2 = mask.copy()
    m2[m2 == E.LOST] = 2
    assert E.psnr(base, off, m2) == pytest.approx(10 * np.log10(255 ** 2 / 256))
    corrupt_known = base.copy()
    corrupt_known[8:, :] += 99.0
    assert E.psnr(base, corrupt_known, mask) == float("inf")
    with pytest.raises(ValueError):
        E.psnr(base, base, np.zeros((10, 10), np.uint8))


def test_csv_layout():
    rows = [E.BenchRow("linescan", 8, 1, 31.123456789, 0.5, 1.0),
            E.BenchRow("optimized", 8, 4, float("inf"), 0.1234567, 4.04999)]
    buf = io.StringIO()
    E.write_csv(rows, buf)
    assert buf.getvalue() == ("order,block_size,threads,psnr_db,seconds,speedup\n"
                              "linescan,8,1,31.123457,0.500000,1.000\n"
                              "optimized,8,4,inf,0.123457,4.050\n")


@pytest.mark.gpu
def test_bench_rows_on_gpu():
    """evalkit.bench through the sm_100a path: linescan at one thread only,
    every optimized thread count, speedup 1 at one thread, PSNRs of the
    concealment (identical across thread counts: the device path does not
    depend on host threads)."""
    y, x = np.mgrid[0:48, 0:48].astype(np.float64)
    img = 120 + 40 * np.sin(x / 5) + 25 * np.cos(y / 7)
    mask = np.zeros((48, 48), np.uint8)
    mask[16:24, 8:16] = 1
    mask[32:40, 24:40] = 1
    from paper_2207_00233_b200 import FseParams

    rows = E.bench(img, mask, block_sizes=(8,), threads=(2, 4),
                   params=FseParams(d=8, iterations=20))
    assert [(r.order, r.threads) for r in rows] == [("linescan", 1), ("optimized", 1), ("optimized", 2),
                                                    ("optimized", 4)]
    assert rows[0].speedup == 1.0 and rows[1].speedup == 1.0
    assert len({r.psnr_db for r in rows[1:]}) == 1 and np.isfinite(rows[1].psnr_db)
    buf = io.StringIO()
    E.write_csv(rows, buf)
    assert buf.getvalue().count("\n") == 5
