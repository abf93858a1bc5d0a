"""Velocity-tuned prediction-filter bank (host-side, built once per stream).

Restates the reference design (/root/reference/pkg/src/clutterwhiten/
design.py): for velocity v the predictor taps are a separable pair of
Dirichlet interpolators re-centred along the motion trajectory through
the group-delay point (design.py:1-16, 109-122); the frequency-domain
coefficients are their unitary DFT on the retained band
|kx| <= Bx, |ky| <= By, all kz (design.py:125-132), stored complex64
(design.py:256-274).  The bank is a constant input of the device kernel
(folded to the half space in cw_api.cu:build_coef); nothing here runs
per frame.

The whole grid is designed in one vectorised pass: the per-velocity tap
cube factors as Dx(mz, mx) * Dy(mz, my), so the three DFTs reduce to two
small batched contractions.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .params import FilterParams, ParamError, validate

__all__ = [
    "dirichlet",
    "SampleKernel",
    "FreqKernel",
    "FilterBank",
    "sample_kernel",
    "kernel_to_freq",
    "build_bank",
    "retained_bin_indices",
]

_POLE_EPS = 1e-9  # design.py:50


def dirichlet(w, order: int):
    """``sin(pi W w) / (W sin(pi w))`` for odd W, with the removable
    singularity at integer w set to its limit 1 (design.py:53-69)."""
    if order < 1 or order % 2 == 0:
        raise ValueError(f"order must be odd and >= 1, got {order}")
    w = np.asarray(w, dtype=np.float64)
    s = np.sin(np.pi * w)
    pole = np.abs(s) < _POLE_EPS
    out = np.where(pole, 1.0, np.sin(np.pi * order * w) / np.where(pole, 1.0, order * s))
    return float(out) if out.ndim == 0 else out


@dataclass(frozen=True)
class SampleKernel:
    """Real taps ``taps[mz, my, mx]`` over the backward-indexed window."""

    velocity: tuple[float, float]
    taps: np.ndarray


@dataclass(frozen=True)
class FreqKernel:
    """Complex coefficients ``coeffs[kz+Kz, ky+By, kx+Bx]`` on the retained band."""

    velocity: tuple[float, float]
    coeffs: np.ndarray


def _grid_span_check(params: FilterParams, vx: float, vy: float) -> None:
    sx = max(abs(v) for v in params.lag_grid_x)
    sy = max(abs(v) for v in params.lag_grid_y)
    if abs(vx) > sx + 1e-12 or abs(vy) > sy + 1e-12:
        raise ParamError(
            f"velocity ({vx}, {vy}) outside the configured grid span (+-{sx}, +-{sy})"
        )


def _axis_interp(m_len: int, order: int, mhat: int, mhat_z: int, v, mz_len: int):
    """D(v, mz, m) = dirichlet((m - mhat - v (mz - mhat_z)) / M, W) for a
    vector of velocities v: shape (len(v), Mz, M)."""
    v = np.atleast_1d(np.asarray(v, dtype=np.float64))
    m = np.arange(m_len)[None, None, :]
    mz = np.arange(mz_len)[None, :, None]
    return dirichlet((m - mhat - v[:, None, None] * (mz - mhat_z)) / m_len, order)


def sample_kernel(params: FilterParams, velocity) -> SampleKernel:
    """Sample-domain prediction taps for one velocity (design.py:109-122)."""
    vx, vy = float(velocity[0]), float(velocity[1])
    _grid_span_check(params, vx, vy)
    mhx, mhy, mhz = params.mhat
    dx = _axis_interp(params.mx, params.wx, mhx, mhz, vx, params.mz)[0]  # (Mz, Mx)
    dy = _axis_interp(params.my, params.wy, mhy, mhz, vy, params.mz)[0]  # (Mz, My)
    gain = params.wx * params.wy / params.bin_count
    return SampleKernel((vx, vy), gain * dy[:, :, None] * dx[:, None, :])


def _band_phases(m_len: int, half_band: int) -> np.ndarray:
    """exp(-j 2 pi k m / M) for k = -B..B (the conjugated synthesis basis)."""
    k = np.arange(-half_band, half_band + 1)
    return np.conj(np.exp(2j * np.pi * np.outer(k, np.arange(m_len)) / m_len))


def kernel_to_freq(kernel: SampleKernel, params: FilterParams) -> FreqKernel:
    """Unitary DFT of the taps restricted to the retained band (design.py:125-132)."""
    cz = _band_phases(params.mz, params.kz)
    cy = _band_phases(params.my, params.by)
    cx = _band_phases(params.mx, params.bx)
    coeffs = np.einsum("am,bn,co,mno->abc", cz, cy, cx, kernel.taps)
    coeffs /= np.sqrt(params.bin_count)
    return FreqKernel(kernel.velocity, coeffs)


def retained_bin_indices(params: FilterParams) -> np.ndarray:
    """Flat (kz, ky, kx) bin index of every coefficient, in coefficient order
    (design.py:195-205)."""
    kz = np.arange(params.mz)[:, None, None]
    ky = (np.arange(-params.by, params.by + 1) + params.ky)[None, :, None]
    kx = (np.arange(-params.bx, params.bx + 1) + params.kx)[None, None, :]
    return ((kz * params.my + ky) * params.mx + kx).reshape(-1).astype(np.int64)


@dataclass
class FilterBank:
    """Per-velocity FreqKernel coefficients, ``coeffs[iy, ix]`` complex64
    (design.py:208-253)."""

    params: FilterParams
    lag_x: np.ndarray
    lag_y: np.ndarray
    coeffs: np.ndarray
    build_seconds: float = 0.0
    retained: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        if self.retained is None:
            self.retained = retained_bin_indices(self.params)

    @property
    def size(self) -> int:
        return len(self.lag_x) * len(self.lag_y)

    @property
    def coeffs_flat(self) -> np.ndarray:
        """(Ly, Lx, retained_count) view."""
        return self.coeffs.reshape(self.coeffs.shape[0], self.coeffs.shape[1], -1)

    def index_of(self, velocity) -> tuple[int, int]:
        """Grid indices (ix, iy) of an exact grid velocity, else ParamError."""
        vx, vy = float(velocity[0]), float(velocity[1])
        hit_x = np.flatnonzero(np.abs(self.lag_x - vx) < 1e-9)
        hit_y = np.flatnonzero(np.abs(self.lag_y - vy) < 1e-9)
        if hit_x.size != 1 or hit_y.size != 1:
            raise ParamError(f"velocity ({vx}, {vy}) is not on the configured velocity grid")
        return int(hit_x[0]), int(hit_y[0])

    def kernel(self, ix: int, iy: int) -> FreqKernel:
        return FreqKernel((float(self.lag_x[ix]), float(self.lag_y[iy])), self.coeffs[iy, ix])


def build_bank(params: FilterParams) -> FilterBank:
    """Design all Ly x Lx predictors (289 by default) in one batched pass."""
    validate(params)
    t0 = time.perf_counter()
    lag_x = np.asarray(params.lag_grid_x, dtype=np.float64)
    lag_y = np.asarray(params.lag_grid_y, dtype=np.float64)
    mhx, mhy, mhz = params.mhat
    dx = _axis_interp(params.mx, params.wx, mhx, mhz, lag_x, params.mz)  # (Lx, Mz, Mx)
    dy = _axis_interp(params.my, params.wy, mhy, mhz, lag_y, params.mz)  # (Ly, Mz, My)
    cz = _band_phases(params.mz, params.kz)
    cy = _band_phases(params.my, params.by)
    cx = _band_phases(params.mx, params.bx)
    gain = params.wx * params.wy / params.bin_count
    # per-velocity spatial transforms, then the temporal DFT over mz
    fx = np.einsum("co,xmo->xmc", cx, dx)          # (Lx, Mz, Wx)
    fy = np.einsum("bn,ymn->ymb", cy, dy)          # (Ly, Mz, Wy)
    coeffs = np.einsum("am,ymb,xmc->yxabc", cz, fy, fx) * (gain / np.sqrt(params.bin_count))
    return FilterBank(
        params=params,
        lag_x=lag_x,
        lag_y=lag_y,
        coeffs=coeffs.astype(np.complex64),
        build_seconds=time.perf_counter() - t0,
    )
