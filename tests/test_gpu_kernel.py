"""Per-window operator on the GPU (fse_run_windows through the run_fse shim)
against the reference's golden vectors and the oracle.  Mirrors the kernel
tests of the reference (test_fse.py:106-319, test_acceptance.py C4/C5)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2207_00233_b200")


def canon(picks, shape):
    return O.canonical_picks(picks, shape)


def test_run_fse_matches_reference_golden(golden):
    g = golden("run_fse_cases.npz")
    for i in range(int(g["n_cases"])):
        v, w = g[f"c{i}_values"], g[f"c{i}_weights"]
        it, gam = int(g[f"c{i}_meta"][0]), float(g[f"c{i}_meta"][1])
        rc = g[f"c{i}_coeff"]
        want = [tuple(x) for x in g[f"c{i}_canon"].tolist()]
        if v.shape[0] >= 128:  # energy trace does not fit shared memory at F=128 fp64
            m, n = P.fse._crop_extent(w)
            out = P.run_fse_batch(v[None, :m, :n], w[None, :m, :n], it, gam, fft_size=v.shape)
            assert canon(out["picks"][0], v.shape) == want, i
            coeff = P.fse.replay_coeff(out["picks"][0], out["plog"][0], v.shape, gam)
            assert np.max(np.abs(coeff - rc)) <= 1e-9 * np.max(np.abs(rc)), i
            continue
        coeff, picks, en, res = P.run_fse(v, w, it, gam)
        assert canon(picks, v.shape) == want, i
        assert np.max(np.abs(coeff - rc)) <= 1e-9 * np.max(np.abs(rc)), i
        assert np.max(np.abs(en - g[f"c{i}_energies"])) <= 1e-9 * g[f"c{i}_energies"][0], i
        assert np.max(np.abs(res - g[f"c{i}_residual"])) <= 1e-9 * 255.0, i


@pytest.mark.parametrize("seed", range(8))
def test_kernel_matches_oracle_random_shapes(seed):
    # test_fse.py:106-129 shapes: generic (non power-of-two) DFT sizes
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(4, 20)), int(rng.integers(4, 20))
    v = rng.uniform(0.0, 255.0, (m, n))
    w = rng.uniform(0.0, 1.0, (m, n))
    w[rng.uniform(size=(m, n)) < 0.35] = 0.0
    w[m // 2, n // 2] = 1.0
    coeff, picks, en, res = P.run_fse(v, w, 25, 0.5)
    rc, rp, re, rr = O.run_fse_c(v, w, 25, 0.5)
    assert canon(picks, (m, n)) == canon(rp, (m, n))
    assert np.max(np.abs(coeff - rc)) <= 1e-9 * np.max(np.abs(rc))
    assert np.max(np.abs(res - rr)) <= 1e-9 * np.max(np.abs(v))
    assert np.max(np.abs(en - re)) <= 1e-9 * re[0]


@pytest.mark.parametrize("F,msz", [(32, 30), (64, 32), (64, 18), (128, 36)])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_batched_windows_fast_path_vs_oracle(F, msz, precision):
    rng = np.random.default_rng(F + msz)
    n = 6
    vals = rng.uniform(0, 255, (n, msz, msz))
    wts = rng.uniform(0, 1, (n, msz, msz)) * (rng.uniform(size=(n, msz, msz)) > 0.2)
    out = P.run_fse_batch(vals, wts, 40, 0.5, precision=precision, fft_size=F)
    for k in range(n):
        vp = np.zeros((F, F)); wp = np.zeros((F, F))
        vp[:msz, :msz] = vals[k]; wp[:msz, :msz] = wts[k]
        rc, rp, _, _ = O.run_fse_c(vp, wp, 40, 0.5)
        coeff = P.fse.replay_coeff(out["picks"][k], out["plog"][k], (F, F), 0.5)
        if precision == "fp64":
            assert canon(out["picks"][k], (F, F)) == canon(rp, (F, F))
            assert np.max(np.abs(coeff - rc)) <= 1e-9 * np.max(np.abs(rc))
        else:
            syn = (np.fft.ifft2(coeff) * F * F).real[:msz, :msz]
            ref = (np.fft.ifft2(rc) * F * F).real[:msz, :msz]
            assert np.max(np.abs(syn - ref)) < 0.5


@settings(max_examples=25, deadline=None)
@given(m=st.integers(2, 12), n=st.integers(2, 12), gamma=st.floats(0.05, 1.0),
       seed=st.integers(0, 2**31 - 1))
def test_energy_never_increases(m, n, gamma, seed):
    rng = np.random.default_rng(seed)
    v = rng.uniform(-100.0, 355.0, (m, n))
    w = rng.uniform(0.0, 1.0, (m, n))
    w[0, 0] = 0.5
    _, _, en, _ = P.run_fse(v, w, 30, gamma)
    assert np.all(np.diff(en) <= 1e-12 * en[0])


def test_c4_energy_monotone_48x48_200_iterations():
    rng = np.random.default_rng(7)
    params = P.FseParams()
    for _ in range(50):
        v = rng.uniform(0.0, 255.0, (48, 48))
        cls = np.full((48, 48), P.AREA_A, dtype=np.uint8)
        r, c = int(rng.integers(0, 33)), int(rng.integers(0, 33))
        cls[r:r + 16, c:c + 16] = P.AREA_BI
        cls[rng.uniform(size=(48, 48)) < 0.15] = P.AREA_R
        w = P.weight_plane((48, 48), cls, params)
        _, _, en, _ = P.run_fse(v, w, 200, params.gamma)
        assert np.all(np.diff(en) <= 1e-12 * en[0])


def test_c5_span_recovery():
    m = n = 48
    params = P.FseParams()
    w = P.weight_plane((m, n), np.full((m, n), P.AREA_A, dtype=np.uint8), params)
    gm, gn = np.arange(m)[:, None], np.arange(n)[None, :]

    def pair(k, amp, ph):
        return 2.0 * (amp * np.exp(1j * ph) * np.exp(2j * np.pi * (k[0] * gm / m + k[1] * gn / n))).real

    v = 80.0 + pair((3, 5), 40.0, 0.7) + pair((7, 2), 25.0, -1.3)
    _, picks, en, _ = P.run_fse(v, w, 100, params.gamma)
    assert en[-1] <= 1e-9 * en[0]
    _, picks, en, _ = P.run_fse(v, w, 60, params.gamma)
    assert {(int(a), int(b)) for a, b in picks} <= {(0, 0), (3, 5), (45, 43), (7, 2), (41, 46)}


def test_residual_initial_energy_and_zero_iterations():
    rng = np.random.default_rng(5)
    v = rng.uniform(0.0, 255.0, (8, 8))
    w = np.zeros((8, 8)); w[2:5, 2:5] = 1.0
    coeff, picks, en, res = P.run_fse(v, w, 0, 0.5)
    assert en[0] == pytest.approx(float((v[2:5, 2:5] ** 2).sum()))
    assert picks.shape == (0, 2) and not coeff.any()


def test_generate_model_api():
    rng = np.random.default_rng(9)
    values = rng.uniform(0, 255, (20, 20))
    cls = np.full((20, 20), P.AREA_A, dtype=np.uint8)
    cls[8:12, 8:12] = P.AREA_BI
    win = P.Window(origin=(0, 0), cls=cls, block_rect=(8, 12, 8, 12), values=values)
    params = P.FseParams(iterations=40, block_size=4)
    model = P.generate_model(win, params)
    assert model.energies.shape == (41,)
    grid = np.zeros((20, 20), dtype=complex)
    for (a, b), c in model.coeffs.items():
        grid[a, b] = c
    np.testing.assert_allclose((np.fft.ifft2(grid) * 400).real, model.synthesized, atol=1e-9)
    np.testing.assert_array_equal(grid, np.conj(grid[np.ix_((20 - np.arange(20)) % 20,
                                                             (20 - np.arange(20)) % 20)]))
    blk = P.extrapolate_block(win, params)
    np.testing.assert_array_equal(blk, model.synthesized[8:12, 8:12])
    # oracle agreement of the block model
    ob = O.extrapolate(values, cls, (8, 12, 8, 12), O.Params(iterations=40, block_size=4), "c")
    assert np.max(np.abs(ob - blk)) < 1e-6
    z = P.generate_model(win, P.FseParams(iterations=0))
    assert z.coeffs == {} and (z.synthesized == 0).all()
    dead = P.Window(origin=(0, 0), cls=np.full((8, 8), P.AREA_BI, np.uint8), block_rect=(0, 8, 0, 8),
                    values=np.zeros((8, 8)))
    with pytest.raises(P.DegenerateWindowError):
        P.generate_model(dead, P.FseParams(iterations=5))


def test_backend_switch():
    assert P.get_backend() == "cuda"
    P.set_backend("cuda")
    with pytest.raises(ValueError):
        P.set_backend("python")
