"""The oracle (oracle/) pinned against the golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from helpers import conceal_case
from oracle import oracle as O


def test_c_oracle_matches_reference_run_fse(golden):
    g = golden("run_fse_cases.npz")
    for i in range(int(g["n_cases"])):
        v, w = g[f"c{i}_values"], g[f"c{i}_weights"]
        it, gam = g[f"c{i}_meta"]
        coeff, picks, en, res = O.run_fse_c(v, w, int(it), float(gam))
        assert O.canonical_picks(picks, v.shape) == [tuple(x) for x in g[f"c{i}_canon"].tolist()], i
        rc = g[f"c{i}_coeff"]
        assert np.max(np.abs(coeff - rc)) <= 1e-9 * np.max(np.abs(rc)), i
        assert np.max(np.abs(en - g[f"c{i}_energies"])) <= 1e-9 * g[f"c{i}_energies"][0], i
        assert np.max(np.abs(res - g[f"c{i}_residual"])) <= 1e-9 * 255.0, i


def test_ref_kernel_build_is_the_golden_kernel(golden):
    k = O.ref_kernel()
    if k is None:
        pytest.skip("oracle/_ref not built (needs /root/reference; oracle/build_ref.sh)")
    g = golden("run_fse_cases.npz")
    for i in range(int(g["n_cases"])):
        it, gam = g[f"c{i}_meta"]
        coeff, picks, en, res = k.run_fse(g[f"c{i}_values"], g[f"c{i}_weights"], int(it), float(gam))
        np.testing.assert_array_equal(picks, g[f"c{i}_picks"])
        np.testing.assert_allclose(coeff, g[f"c{i}_coeff"], rtol=0, atol=1e-12 * np.abs(coeff).max())


def test_weight_plane_matches_reference(golden):
    g = golden("weight_cases.npz")
    for i in range(int(g["n_cases"])):
        cls = g[f"w{i}_cls"]
        got = O.weight_plane(cls.shape, cls, 0.8, 0.2)
        np.testing.assert_allclose(got, g[f"w{i}_plane"], rtol=1e-15, atol=0)


def test_weight_known_answers():
    # test_fse.py:59-65 closed forms
    cls = np.zeros((9, 9), np.uint8)
    plane = O.weight_plane((9, 9), cls, 0.8, 0.2)
    assert plane[4, 4] == 1.0
    assert plane[4, 5] == pytest.approx(0.8)
    assert plane[3, 3] == pytest.approx(0.8 ** np.sqrt(2.0))
    np.testing.assert_allclose(O.weight_plane((9, 9), np.full((9, 9), 3, np.uint8), 0.8, 0.2),
                               0.2 * plane, rtol=0, atol=0)


def test_oracle_schedule_matches_reference(golden):
    g = golden("schedule_cases.npz")
    for i in range(int(g["n_cases"])):
        t = g[f"s{i}_table"]
        grid = O.Grid.of(t.shape[0] * 4, t.shape[1] * 4, 4)
        c = O.init_counts(grid, t)
        np.testing.assert_array_equal(c, g[f"s{i}_counts"])
        ptr, bl = g[f"s{i}_ptr"], g[f"s{i}_blocks"]
        if t.size > 4096:
            continue  # the pure-Python restatement is slow on the big grids
        assert O.schedule_all(grid, c) == [bl[ptr[k]:ptr[k + 1]].tolist() for k in range(len(ptr) - 1)]


@pytest.mark.parametrize("i", range(11))
def test_oracle_conceal_matches_reference(golden, i):
    g = golden("conceal_cases.npz")
    c = conceal_case(g, i)
    if c["iterations"] * c["processed"] > 8000 and c["fft"] == (128, 128):
        pytest.skip("large case covered by the GPU suite")
    p = O.Params(d=c["d"], rho=c["rho"], delta=c["delta"], gamma=c["gamma"],
                 iterations=c["iterations"], block_size=c["block_size"], fft_size=c["fft"])
    img, msk, rep = O.conceal(c["image"], c["mask"], p, c["order"], kernel="c", want_picks=True)
    np.testing.assert_array_equal(msk, c["out_mask"])
    assert rep.batches == c["batches"]
    assert rep.unconcealed_blocks == c["unconcealed"]
    assert np.max(np.abs(img - c["out_image"])) <= 1e-9
    F = c["fft"] or None
    for b, pk in zip(c["pick_blocks"].tolist(), c["picks"]):
        shape = F if F else None
        if shape is None:
            continue  # native DFT sizes vary per window; covered by the sample check
        assert O.canonical_picks(rep.picks[b], shape) == [tuple(x) for x in pk.tolist()]
