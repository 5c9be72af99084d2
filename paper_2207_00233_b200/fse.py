"""FSE model parameters and the per-window operator (B200 device path).

Mirrors fsefill.fse (/root/reference/pkg/src/fsefill/fse.py): FseParams,
DegenerateWindowError, Model, weight_plane, weight, dft_basis, generate_model,
extrapolate_block and the backend switch.  The model fit itself
(``run_fse``, reference ``_kernel.pyx:128-187``) runs on the GPU through
``fse_run_windows`` of libfse_b200; the only backend is ``"cuda"`` — there is
no CPU fallback.

Additions over the reference:
  * ``FseParams.fft_size``: None keeps the reference's DFT size (the window
    shape, fse.py:158-159); an int F or a pair (F1, F2) zero-pads every window
    at the top-left to that DFT size (BASELINE.json's "FFT 64x64" etc.).
  * ``precision``: "fp64" (reference arithmetic type) or "fp32".
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grid import AREA_A, AREA_R, Window

PRECISIONS = ("fp64", "fp32")
_active = "cuda"
_BACKENDS = ("cuda",)


def get_backend() -> str:
    return _active


def set_backend(name: str) -> None:
    """Only the CUDA backend exists (fse.py:37-44 contract: ValueError otherwise)."""
    if name not in _BACKENDS:
        raise ValueError(f"backend {name!r} not available (have: {sorted(_BACKENDS)})")


class DegenerateWindowError(ValueError):
    """A window with no positively weighted sample (fse.py:51-52)."""


@dataclass(frozen=True)
class FseParams:
    """fse.py:55-86 plus ``fft_size`` (see module docstring)."""

    d: int = 16
    rho: float = 0.8
    delta: float = 0.2
    gamma: float = 0.5
    iterations: int = 200
    block_size: int = 16
    fft_size: int | tuple[int, int] | None = None

    def __post_init__(self):
        if self.d < 0:
            raise ValueError("d must be >= 0")
        if not 0.0 < self.rho < 1.0:
            raise ValueError("rho must lie in (0, 1)")
        if not 0.0 <= self.delta <= 1.0:
            raise ValueError("delta must lie in [0, 1]")
        if not 0.0 < self.gamma <= 1.0:
            raise ValueError("gamma must lie in (0, 1]")
        if self.iterations < 0:
            raise ValueError("iterations must be >= 0")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        if self.fft_size is not None:
            f1, f2 = self.fft_dims((1, 1))
            if f1 < 1 or f2 < 1:
                raise ValueError("fft_size must be positive")

    def fft_dims(self, window_shape) -> tuple[int, int]:
        if self.fft_size is None:
            return int(window_shape[0]), int(window_shape[1])
        if isinstance(self.fft_size, (tuple, list)):
            return int(self.fft_size[0]), int(self.fft_size[1])
        return int(self.fft_size), int(self.fft_size)

    def to_c(self) -> _lib.FseParamsC:
        f1, f2 = (0, 0) if self.fft_size is None else self.fft_dims((0, 0))
        return _lib.FseParamsC(self.d, self.block_size, self.iterations, f1, f2,
                               self.rho, self.delta, self.gamma)


@dataclass
class Model:
    """Fitted window model (fse.py:89-102)."""

    coeffs: dict
    synthesized: np.ndarray
    energies: np.ndarray
    picks: np.ndarray = field(repr=False, default=None)


def weight_plane(shape, classes, params: FseParams) -> np.ndarray:
    """rho^dist on A, delta*rho^dist on R, 0 on BI/BO; distance from the window's
    geometric centre ((M-1)/2, (N-1)/2) (fse.py:105-119)."""
    m, n = shape
    dm = np.arange(m, dtype=np.float64) - (m - 1) / 2.0
    dn = np.arange(n, dtype=np.float64) - (n - 1) / 2.0
    decay = params.rho ** np.sqrt(dm[:, None] ** 2 + dn[None, :] ** 2)
    return np.where(classes == AREA_A, decay,
                    np.where(classes == AREA_R, params.delta * decay, 0.0)).astype(np.float64)


def weight(m: int, n: int, shape, cls: int, params: FseParams) -> float:
    """Scalar twin of weight_plane (fse.py:122-130)."""
    mm, nn = shape
    dist = np.sqrt((m - (mm - 1) / 2.0) ** 2 + (n - (nn - 1) / 2.0) ** 2)
    if cls == AREA_A:
        return float(params.rho ** dist)
    if cls == AREA_R:
        return float(params.delta * params.rho ** dist)
    return 0.0


def dft_basis(shape, k) -> np.ndarray:
    """exp(+j2pi(k1 m/M + k2 n/N)) (fse.py:133-139)."""
    m, n = shape
    return np.outer(np.exp(2j * np.pi * k[0] * np.arange(m) / m),
                    np.exp(2j * np.pi * k[1] * np.arange(n) / n))


def decay_table(rho: float, dim: int) -> np.ndarray:
    """decay[i, j] = rho ** sqrt((i/2)^2 + (j/2)^2) for doubled centre offsets
    i = |2m - (M-1)|, j = |2n - (N-1)|: the same float64 expression as
    fse.py:112-115, tabulated once for every window shape."""
    h = np.arange(dim, dtype=np.float64) / 2.0
    return np.ascontiguousarray(rho ** np.sqrt(h[:, None] ** 2 + h[None, :] ** 2))


# --------------------------------------------------------------- device operator

def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2207_00233_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _dtype(precision: str):
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    torch = _torch()
    return (torch.float64, _lib.FSE_F64) if precision == "fp64" else (torch.float32, _lib.FSE_F32)


def replay_coeff(picks, plog, shape, gamma: float) -> np.ndarray:
    """Coefficient grid from the device's pick log, accumulated exactly as
    _kernel.pyx:50-71 does (c[a,b] += gamma*p, c[-a,-b] += gamma*conj(p);
    gamma*Re(p) alone for self-conjugate picks)."""
    m, n = shape
    c_re = np.zeros((m, n))
    c_im = np.zeros((m, n))
    g = float(gamma)
    for (a, b), (pr, pi) in zip(np.asarray(picks).tolist(), np.asarray(plog, dtype=np.float64).tolist()):
        if (2 * a) % m == 0 and (2 * b) % n == 0:
            c_re[a, b] += g * pr
        else:
            ta, tb = (m - a) % m, (n - b) % n
            c_re[a, b] += g * pr
            c_im[a, b] += g * pi
            c_re[ta, tb] += g * pr
            c_im[ta, tb] -= g * pi
    return c_re + 1j * c_im


def run_fse_batch(values, weights, iterations: int, gamma: float, precision: str = "fp64",
                  fft_size=None, debug: bool = False):
    """Batched device model fit of n windows [n, M, N] zero-padded to fft_size.

    Returns dict with picks (n, I, 2) int32, plog (n, I, 2) float64 and, with
    debug=True, energies (n, I+1) and residual (n, F1, F2)."""
    torch = _torch()
    tdt, code = _dtype(precision)
    v = torch.as_tensor(np.ascontiguousarray(values), dtype=tdt).cuda()
    w = torch.as_tensor(np.ascontiguousarray(weights), dtype=tdt).cuda()
    if v.dim() != 3 or v.shape != w.shape:
        raise ValueError("values/weights must be [n, M, N] and equal shapes")
    n, M, N = v.shape
    if fft_size is None:
        F1, F2 = M, N
    elif isinstance(fft_size, (tuple, list)):
        F1, F2 = int(fft_size[0]), int(fft_size[1])
    else:
        F1 = F2 = int(fft_size)
    it = int(iterations)
    picks = torch.zeros((n, max(it, 1), 2), dtype=torch.int32, device="cuda")
    plog = torch.zeros((n, max(it, 1), 2), dtype=tdt, device="cuda")
    en = res = None
    if debug:
        en = torch.zeros((n, it + 1), dtype=tdt, device="cuda")
        res = torch.zeros((n, F1, F2), dtype=tdt, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().fse_run_windows(
        n, M, N, F1, F2, v.data_ptr(), w.data_ptr(), it, float(gamma), code,
        picks.data_ptr(), plog.data_ptr(),
        en.data_ptr() if debug else None, res.data_ptr() if debug else None, stream))
    torch.cuda.synchronize()
    out = {"picks": picks[:, :it].cpu().numpy(), "plog": plog[:, :it].double().cpu().numpy()}
    if debug:
        out["energies"] = en.double().cpu().numpy()
        out["residual"] = res.double().cpu().numpy()
    return out


def _crop_extent(weights: np.ndarray) -> tuple[int, int]:
    """Smallest top-left M x N holding every positive weight (the rest of the plane
    contributes nothing; the DFT size keeps the full shape)."""
    rows = np.flatnonzero((weights > 0).any(axis=1))
    cols = np.flatnonzero((weights > 0).any(axis=0))
    if rows.size == 0:
        return 1, 1
    return int(rows[-1]) + 1, int(cols[-1]) + 1


def run_fse(values, weights, iterations: int, gamma: float, precision: str = "fp64"):
    """Drop-in for fsefill._kernel.run_fse (contract _kernel_py.py:13-30):
    returns (coeff c128[M,N], picks i32[I,2], energies f64[I+1], residual f64[M,N]).
    The DFT size is the input shape, as in the reference."""
    values = np.ascontiguousarray(values, dtype=np.float64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    m, n = values.shape
    cm, cn = _crop_extent(weights)
    out = run_fse_batch(values[None, :cm, :cn], weights[None, :cm, :cn], iterations, gamma,
                        precision=precision, fft_size=(m, n), debug=True)
    coeff = replay_coeff(out["picks"][0], out["plog"][0], (m, n), gamma)
    return coeff, out["picks"][0].astype(np.int32), out["energies"][0], out["residual"][0]


def generate_model(win: Window, params: FseParams, precision: str = "fp64") -> Model:
    """fse.py:142-169 on the device kernel; synthesis = Re(ifft2(coeff) * F1 F2)
    over the (padded) DFT plane, cut to the window."""
    values = np.ascontiguousarray(win.values, dtype=np.float64)
    weights = weight_plane(values.shape, win.cls, params)
    if not (weights > 0.0).any():
        raise DegenerateWindowError("window has no usable samples")
    m, n = values.shape
    F1, F2 = params.fft_dims((m, n))
    if F1 < m or F2 < n:
        raise ValueError(f"fft_size {(F1, F2)} smaller than the window {(m, n)}")
    cm, cn = _crop_extent(weights)
    try:
        out = run_fse_batch(values[None, :cm, :cn], weights[None, :cm, :cn], params.iterations,
                            params.gamma, precision=precision, fft_size=(F1, F2), debug=True)
        energies = out["energies"][0]
    except _lib.FseUnsupported:  # energy trace does not fit in shared memory at this size
        out = run_fse_batch(values[None, :cm, :cn], weights[None, :cm, :cn], params.iterations,
                            params.gamma, precision=precision, fft_size=(F1, F2), debug=False)
        energies = np.full(params.iterations + 1, np.nan)
    picks = out["picks"][0].astype(np.int32)
    coeff = replay_coeff(picks, out["plog"][0], (F1, F2), params.gamma)
    synthesized = (np.fft.ifft2(coeff) * (F1 * F2)).real[:m, :n]
    coeffs = {}
    for a, b in picks.tolist():
        coeffs[(a, b)] = complex(coeff[a, b])
        pa, pb = (F1 - a) % F1, (F2 - b) % F2
        coeffs[(pa, pb)] = complex(coeff[pa, pb])
    return Model(coeffs=coeffs, synthesized=synthesized, energies=energies, picks=picks)


def extrapolate_block(win: Window, params: FseParams, precision: str = "fp64") -> np.ndarray:
    """Model values over the window's block (fse.py:172-176)."""
    model = generate_model(win, params, precision)
    r0, r1, c0, c1 = win.block_rect
    return model.synthesized[r0:r1, c0:c1].copy()
