"""TEST INFRASTRUCTURE ONLY -- the float64 CPU oracle (parity checker).

Python driver for ``libcw_oracle.so`` (``cw_oracle.c``), a float64
restatement of the reference ``clutterwhiten`` per-pixel pipeline.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this module; the product path never does.

The phase tables, gains and the filter bank are rebuilt here with numpy
exactly as the reference builds them, so the C kernels see bit-identical
inputs:

* ``_axis_tables``      -- /root/reference/pkg/src/clutterwhiten/spectrum.py:65-74
* ``_autocorr_tables``  -- flow.py:87-97
* ``pick_gains``        -- flow.py:147-163
* ``dirichlet``         -- design.py:53-69
* ``sample_kernel``     -- design.py:109-122
* ``kernel_to_freq``    -- design.py:125-132 (+ ``_band_table`` 135-139)
* ``build_bank``        -- design.py:256-274 (complex64 storage)
* ``retained_bin_indices`` -- design.py:195-205
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libcw_oracle.so")
_lib = None


def build() -> str:
    """Compile the C oracle in place (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    dp = ctypes.POINTER(ctypes.c_double)
    lib.cwo_create.restype = ctypes.c_void_p
    lib.cwo_create.argtypes = [
        ctypes.POINTER(ctypes.c_int), ctypes.c_double,
        ctypes.c_int, dp, ctypes.c_int, dp,
        dp, dp, dp, dp, dp, dp, dp, dp,
        ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
    ]
    lib.cwo_destroy.argtypes = [ctypes.c_void_p]
    lib.cwo_set_threads.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.cwo_push.restype = ctypes.c_int
    lib.cwo_push.argtypes = [
        ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float),
        ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int32), dp, dp,
        ctypes.POINTER(ctypes.c_longlong), ctypes.c_int, ctypes.c_int, dp,
    ]
    lib.cwo_sbins.restype = dp
    lib.cwo_sbins.argtypes = [ctypes.c_void_p]
    lib.cwo_rhat.restype = dp
    lib.cwo_rhat.argtypes = [ctypes.c_void_p]
    _lib = lib
    return lib


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


# -- reference tables (restated) ---------------------------------------------


def axis_tables(p):
    """spectrum.py:65-74: e[ik, m] = exp(+j2pi k m / M), k = -K..K."""
    out = []
    for m_len in (2 * p.kx + 1, 2 * p.ky + 1, 2 * p.kz + 1):
        k = np.arange(m_len) - (m_len - 1) // 2
        m = np.arange(m_len)
        out.append(np.exp(2j * np.pi * np.outer(k, m) / m_len))
    return tuple(out)


def autocorr_tables(p):
    """flow.py:87-97."""
    mx, my, mz = 2 * p.kx + 1, 2 * p.ky + 1, 2 * p.kz + 1
    kz = np.arange(mz) - p.kz
    az = np.exp(-2j * np.pi * kz / mz)
    kx = np.arange(mx) - p.kx
    ky = np.arange(my) - p.ky
    lag_x = np.asarray(p.lag_grid_x, dtype=np.float64)
    lag_y = np.asarray(p.lag_grid_y, dtype=np.float64)
    axl = np.exp(-2j * np.pi * np.outer(lag_x, kx) / mx)
    ayl = np.exp(-2j * np.pi * np.outer(lag_y, ky) / my)
    return az, axl, ayl


def pick_gains(p):
    """flow.py:147-163: A(0)/A(l) per axis, A(l) = 1/4 + cos(2 pi l / M)/8."""
    lag_x = np.asarray(p.lag_grid_x, dtype=np.float64)
    lag_y = np.asarray(p.lag_grid_y, dtype=np.float64)
    ax = 0.25 + 0.125 * np.cos(2.0 * np.pi * lag_x / (2 * p.kx + 1))
    ay = 0.25 + 0.125 * np.cos(2.0 * np.pi * lag_y / (2 * p.ky + 1))
    return 0.375 / ax, 0.375 / ay


def dirichlet(w, order):
    """design.py:53-69: periodic sinc with the integer-w limit set to 1."""
    w = np.asarray(w, dtype=np.float64)
    den = order * np.sin(np.pi * w)
    num = np.sin(np.pi * order * w)
    near_pole = np.abs(np.sin(np.pi * w)) < 1e-9
    safe = np.where(near_pole, 1.0, den)
    return np.where(near_pole, 1.0, num / safe)


def sample_taps(p, vx, vy):
    """design.py:109-122."""
    mx, my, mz = 2 * p.kx + 1, 2 * p.ky + 1, 2 * p.kz + 1
    wx, wy = 2 * p.bx + 1, 2 * p.by + 1
    mhx, mhy, mhz = p.mhat
    ax = np.arange(mx).reshape(1, 1, mx)
    ay = np.arange(my).reshape(1, my, 1)
    az = np.arange(mz).reshape(mz, 1, 1)
    gain = wx * wy / (mx * my * mz)
    return (
        gain
        * dirichlet((ax - mhx - vx * (az - mhz)) / mx, wx)
        * dirichlet((ay - mhy - vy * (az - mhz)) / my, wy)
    )


def _band_table(m_len, half_band):
    """design.py:135-139."""
    k = np.arange(-half_band, half_band + 1)
    m = np.arange(m_len)
    return np.exp(2j * np.pi * np.outer(k, m) / m_len)


def bank_coeffs(p):
    """design.py:125-132 + 256-274: (Ly, Lx, Mz, Wy, Wx) complex64."""
    mx, my, mz = 2 * p.kx + 1, 2 * p.ky + 1, 2 * p.kz + 1
    nb = mx * my * mz
    cz = np.conj(_band_table(mz, p.kz))
    cy = np.conj(_band_table(my, p.by))
    cx = np.conj(_band_table(mx, p.bx))
    lag_x = np.asarray(p.lag_grid_x, dtype=np.float64)
    lag_y = np.asarray(p.lag_grid_y, dtype=np.float64)
    out = np.empty((len(lag_y), len(lag_x), mz, 2 * p.by + 1, 2 * p.bx + 1), np.complex64)
    for iy, vy in enumerate(lag_y):
        for ix, vx in enumerate(lag_x):
            c = np.einsum("am,bn,co,mno->abc", cz, cy, cx, sample_taps(p, vx, vy))
            c /= np.sqrt(nb)
            out[iy, ix] = c.astype(np.complex64)
    return out


def retained_bin_indices(p):
    """design.py:195-205: flat (kz, ky, kx) bin index per coefficient."""
    mx, my = 2 * p.kx + 1, 2 * p.ky + 1
    idx = []
    for ikz in range(2 * p.kz + 1):
        for ky in range(-p.by, p.by + 1):
            for kx in range(-p.bx, p.bx + 1):
                idx.append((ikz * my + ky + p.ky) * mx + kx + p.kx)
    return np.asarray(idx, dtype=np.int64)


# -- the oracle pipeline -------------------------------------------------------


class OraclePipeline:
    """float64 CPU restatement of ``Pipeline`` (pipeline.py:102-305).

    ``params`` is any object with the FilterParams attributes (the product's
    or the reference's).  ``process_frame`` returns ``None`` during warm-up,
    else a dict with ``frame_index, residual, prediction, indices,
    velocities, imag_peak`` (the WhitenedOutput fields).
    """

    def __init__(self, params, width, height, threads=None, forced_velocity=None, bank=None):
        lib = _load()
        p = params
        self.params = p
        self.width, self.height = int(width), int(height)
        mx, my, mz = 2 * p.kx + 1, 2 * p.ky + 1, 2 * p.kz + 1
        if width < mx or height < my:
            raise ValueError("image smaller than analysis window")
        self.threads = int(threads or os.cpu_count() or 1)
        ex, ey, ez = axis_tables(p)
        az, axl, ayl = autocorr_tables(p)
        gx, gy = pick_gains(p)
        self.lag_x = np.ascontiguousarray(p.lag_grid_x, dtype=np.float64)
        self.lag_y = np.ascontiguousarray(p.lag_grid_y, dtype=np.float64)
        if bank is None:
            bank = bank_coeffs(p)
        bank = np.ascontiguousarray(np.asarray(bank, dtype=np.complex64))
        self._bank = bank.reshape(len(self.lag_y), len(self.lag_x), -1)
        self._retained = np.ascontiguousarray(retained_bin_indices(p))
        nc = self._retained.size
        geom = (ctypes.c_int * 11)(p.kx, p.ky, p.kz, p.bx, p.by, *p.mhat, self.width, self.height, self.threads)
        self._keep = [np.ascontiguousarray(t, dtype=np.complex128) for t in (ex, ey, ez, az, axl, ayl)]
        self._keep += [np.ascontiguousarray(g, dtype=np.float64) for g in (gx, gy)]
        tables = [_ptr(t.view(np.float64), ctypes.c_double) for t in self._keep[:6]]
        gains = [_ptr(g, ctypes.c_double) for g in self._keep[6:]]
        self._h = lib.cwo_create(
            geom, float(p.alpha), len(self.lag_x), _ptr(self.lag_x, ctypes.c_double),
            len(self.lag_y), _ptr(self.lag_y, ctypes.c_double), *tables, *gains,
            _ptr(self._bank.view(np.float32), ctypes.c_float), _ptr(self._retained, ctypes.c_int64), nc,
        )
        if not self._h:
            raise MemoryError("oracle allocation failed")
        self._forced = (-1, -1)
        if forced_velocity is not None:
            ix = int(np.nonzero(np.abs(self.lag_x - forced_velocity[0]) < 1e-9)[0][0])
            iy = int(np.nonzero(np.abs(self.lag_y - forced_velocity[1]) < 1e-9)[0][0])
            self._forced = (ix, iy)
        self.last_timings = {}

    def set_threads(self, n):
        self.threads = int(n)
        _load().cwo_set_threads(self._h, self.threads)

    def process_frame(self, frame):
        lib = _load()
        frame = np.ascontiguousarray(frame, dtype=np.float32)
        if frame.shape != (self.height, self.width):
            raise ValueError(f"frame shape {frame.shape} != {(self.height, self.width)}")
        h, w = self.height, self.width
        res = np.zeros((h, w), np.float32)
        pred = np.zeros((h, w), np.float32)
        idx = np.zeros((h, w, 2), np.int32)
        vel = np.zeros((h, w, 2), np.float64)
        peak = ctypes.c_double(0.0)
        fidx = ctypes.c_longlong(0)
        tim = np.zeros(4, np.float64)
        t0 = time.perf_counter()
        ready = lib.cwo_push(
            self._h, _ptr(frame, ctypes.c_float), _ptr(res, ctypes.c_float), _ptr(pred, ctypes.c_float),
            _ptr(idx, ctypes.c_int32), _ptr(vel, ctypes.c_double), ctypes.byref(peak), ctypes.byref(fidx),
            self._forced[0], self._forced[1], _ptr(tim, ctypes.c_double),
        )
        self.last_timings = {
            "spectrum": tim[0], "conditioning": tim[1], "autocorr": tim[2], "filtering": tim[3],
            "pipeline": time.perf_counter() - t0,
        }
        if not ready:
            return None
        return {
            "frame_index": int(fidx.value), "residual": res, "prediction": pred,
            "indices": idx, "velocities": vel, "imag_peak": float(peak.value),
        }

    def sbins(self):
        """Current (H, W, Mz, My, Mx) complex128 spectrum (copy)."""
        p = self.params
        n = self.height * self.width * (2 * p.kx + 1) * (2 * p.ky + 1) * (2 * p.kz + 1)
        buf = np.ctypeslib.as_array(_load().cwo_sbins(self._h), shape=(2 * n,)).copy()
        return buf.view(np.complex128).reshape(
            self.height, self.width, 2 * p.kz + 1, 2 * p.ky + 1, 2 * p.kx + 1)

    def rhat(self):
        """Current smoothed autocorrelation (H, W, Ly, Lx) float64 (copy)."""
        n = self.height * self.width * len(self.lag_x) * len(self.lag_y)
        buf = np.ctypeslib.as_array(_load().cwo_rhat(self._h), shape=(n,)).copy()
        return buf.reshape(self.height, self.width, len(self.lag_y), len(self.lag_x))

    def close(self):
        if getattr(self, "_h", None):
            _load().cwo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False
