"""Drop-in ``Pipeline`` for the reference whitening path, running on B200.

Mirrors /root/reference/pkg/src/clutterwhiten/pipeline.py: same
constructor (118-127), ``process_frame`` contract (201-294: ``None`` during
the Mz-1 warm-up frames, then a ``WhitenedOutput`` aligned to input index
``n - mhat_z``), properties, context manager and error behaviour.  Each
call uploads the frame and runs ONE fused sm_100a kernel through the C ABI
(include/cw_b200.h); outputs are fresh host arrays per call.

Differences from the reference, by design:
* ``strategy`` is accepted and reported but never changes results (the
  device path has one execution shape).
* ``spectrum_backend="naive"`` (the reference's non-recursive backend,
  spectrum.py:257-327) evaluates every pixel's window DFT directly on the
  GPU (csrc/cw_naive.cuh) and feeds the same fused flow/PEF kernel.
* ``imag_peak`` (max |Im acc|, pipeline.py:293) is evaluated from the
  folded imaginary PEF coefficients: the kernel stores the half spectrum
  (S(-k) = conj S(k) exactly), so Im acc = sum S.re (c.im + c'.im) +
  S.im (c.re - c'.re) over the pairs (k, -k).  For a Hermitian bank (every
  bank ``build_bank`` makes: c(-k) = conj c(k) bit for bit) all those
  coefficients are exactly 0 and so is imag_peak; an injected non-Hermitian
  bank gets it computed from the device spectrum (``process_frame`` only).
* ``last_timings`` has the reference's keys (pipeline.py:210-285); the
  stages run fused in one kernel, so "conditioning", "autocorr" and
  "filtering" are 0.0 and "spectrum" holds the whole call; with
  ``device_timing=True`` "kernel" adds the fused kernel's device time.
"""

from __future__ import annotations

import ctypes
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native
from .design import FilterBank, FreqKernel, build_bank
from .flow import VelocityField
from .parallel import ExecStrategy
from .params import FilterParams, ParamError, validate

__all__ = ["WhitenedOutput", "Pipeline", "apply_pef", "valid_bounds", "valid_mask"]


def valid_bounds(params: FilterParams, width: int, height: int):
    """Inclusive output bounds (ox_lo, ox_hi, oy_lo, oy_hi) with a full
    analysis window behind the anchor (pipeline.py:41-50)."""
    mhx, mhy, _ = params.mhat
    return (params.mx - 1 - mhx, width - 1 - mhx, params.my - 1 - mhy, height - 1 - mhy)


def valid_mask(params: FilterParams, width: int, height: int) -> np.ndarray:
    """(H, W) bool mask of valid output pixels (pipeline.py:53-58)."""
    x0, x1, y0, y1 = valid_bounds(params, width, height)
    mask = np.zeros((height, width), dtype=bool)
    mask[y0 : y1 + 1, x0 : x1 + 1] = True
    return mask


def apply_pef(bins, kernel, delayed_intensity: float):
    """One pixel's prediction/residual from its (Mz, My, Mx) bins
    (host utility, pipeline.py:61-81)."""
    coeffs = kernel.coeffs if isinstance(kernel, FreqKernel) else np.asarray(kernel)
    bins = np.asarray(bins, dtype=np.complex128)
    mz, wy, wx = coeffs.shape
    if bins.ndim != 3 or bins.shape[0] != mz:
        raise ValueError(f"bins shape {bins.shape} incompatible with kernel {coeffs.shape}")
    cy, cx = (bins.shape[1] - 1) // 2, (bins.shape[2] - 1) // 2
    hy, hx = (wy - 1) // 2, (wx - 1) // 2
    band = bins[:, cy - hy : cy + hy + 1, cx - hx : cx + hx + 1]
    pred = float(np.sum(coeffs.astype(np.complex128) * band).real)
    return pred, float(delayed_intensity) - pred


class _LazyVelocityField(VelocityField):
    """VelocityField whose int32 ``indices`` and float64 ``velocities``
    (flow.py:134-144) are expanded from the device's (ix, iy) pairs on first
    access (uint8 pairs through 64K-entry lookup tables; uint16 pairs for
    lag grids longer than 256 directly)."""

    def __init__(self, vidx, pipe):
        self._vidx, self._pipe = vidx, pipe
        self._i = self._v = None

    @property
    def indices(self):
        if self._i is None:
            self._i = self._pipe._indices_of(self._vidx)
        return self._i

    @indices.setter
    def indices(self, value):
        self._i = value

    @property
    def velocities(self):
        if self._v is None:
            self._v = self._pipe._velocities_of(self._vidx)
        return self._v

    @velocities.setter
    def velocities(self, value):
        self._v = value


class _PinnedPool:
    """Recycled page-locked host buffers for per-call output arrays.

    Every ``process_frame`` returns fresh arrays (the reference copies its
    outputs, pipeline.py:288-292); backing them with pinned memory lets the
    device copy them at full PCIe rate.  A buffer goes back to the pool when
    the array handed out (and every view of it) has been garbage collected.
    """

    # pinned bytes handed out at once before further outputs fall back to
    # ordinary (pageable) numpy arrays: callers that keep every residual
    # (cli._cmd_filter appends them all) must not pin unbounded host memory
    MAX_OUTSTANDING_BYTES = 256 << 20

    def __init__(self):
        self._free: dict[tuple, list] = {}
        # re-entrant: _give runs from weakref finalizers, which cyclic GC may
        # fire on this thread while take/take_outputs holds the lock
        self._lock = threading.RLock()
        self._outstanding = 0

    def take_outputs(self, h, w, idx_bytes=1):
        """(residual, prediction, velocity-index) arrays of one call, carved
        from a single pinned block (one allocation / finalizer per call; the
        block returns to the pool when the last of the three is collected)."""
        import torch

        key = ("outputs", h, w, idx_bytes)
        hw = h * w
        nbytes = (8 + 2 * idx_bytes) * hw
        with self._lock:
            if self._outstanding + nbytes > self.MAX_OUTSTANDING_BYTES and self._outstanding > 0:
                tensor = False  # pool exhausted: pageable arrays (the device copies through staging)
            else:
                stack = self._free.setdefault(key, [])
                tensor = stack.pop() if stack else None
                self._outstanding += nbytes
        if tensor is False:
            blk = np.empty(nbytes, np.uint8)
        else:
            if tensor is None:
                tensor = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
            blk = tensor.numpy()
            weakref.finalize(blk, self._give, key, tensor, nbytes)
        res = blk[: 4 * hw].view(np.float32).reshape(h, w)
        pred = blk[4 * hw : 8 * hw].view(np.float32).reshape(h, w)
        vidx = blk[8 * hw :].view(np.uint8 if idx_bytes == 1 else np.uint16).reshape(h, w, 2)
        return res, pred, vidx

    def _give(self, key, tensor, nbytes):
        with self._lock:
            self._free.setdefault(key, []).append(tensor)
            self._outstanding -= nbytes


@dataclass
class WhitenedOutput:
    """One whitened frame (pipeline.py:84-99).

    ``detections`` / ``metrics`` are filled only when the pipeline was built
    with ``detect_threshold`` (the fused final-threshold epilogue):
    detections = (N, 3) float64 [x, y, residual] rows sorted by (y, x);
    metrics = {peak_abs_residual, peak_x, peak_y, residual_rms, n_valid,
    n_detections, truncated} (cli.compute_metrics_row without ground truth).
    """

    frame_index: int
    residual: np.ndarray
    prediction: np.ndarray
    velocity: VelocityField
    mask: np.ndarray
    imag_peak: float
    detections: np.ndarray | None = None
    metrics: dict | None = None


class Pipeline:
    """Streaming whitening filter for one frame geometry on one GPU.

    Parameters are those of the reference (pipeline.py:102-127) plus
    ``device`` (CUDA ordinal).
    """

    def __init__(
        self,
        params: FilterParams,
        width: int,
        height: int,
        strategy: ExecStrategy | str = "serial",
        spectrum_backend: str = "recursive",
        forced_velocity=None,
        bank: FilterBank | None = None,
        device: int = 0,
        detect_threshold: float | None = None,
        max_detections: int = 65536,
        device_timing: bool = False,
        _strip: tuple[int, int] = (0, 0),
    ):
        validate(params)
        if isinstance(strategy, str):
            strategy = ExecStrategy.parse(strategy)
        self._strategy = strategy
        if width < params.mx or height < params.my:
            raise ParamError(
                f"image {width}x{height} smaller than analysis window {params.mx}x{params.my}"
            )
        if spectrum_backend not in ("recursive", "naive"):
            raise ValueError(f"unknown spectrum backend {spectrum_backend!r}")
        self.spectrum_backend = spectrum_backend
        if bank is None:
            bank = build_bank(params)
        elif bank.params != params:
            raise ParamError("filter bank was built for different parameters")
        self.params = params
        self.width = int(width)
        self.height = int(height)
        self.bank = bank
        self.device = int(device)
        self.mask = valid_mask(params, width, height)
        self.mask.setflags(write=False)
        self.last_timings: dict[str, float] = {}
        self._lag_x = np.asarray(params.lag_grid_x, dtype=np.float64)
        self._lag_y = np.asarray(params.lag_grid_y, dtype=np.float64)
        # (ix | iy << 8) -> (ix, iy) int32 and (vx, vy) float64
        code = np.arange(65536)  # (used for grids of <= 256 lags, i.e. uint8 index pairs)
        ix, iy = np.minimum(code & 255, len(self._lag_x) - 1), np.minimum(code >> 8, len(self._lag_y) - 1)
        self._lut_i = np.stack([code & 255, code >> 8], axis=-1).astype(np.int32)
        self._lut_v = np.stack([self._lag_x[ix], self._lag_y[iy]], axis=-1)
        self._pool = _PinnedPool()

        # folded imaginary PEF coefficients c(k).im + c(-k).im, c(k).re - c(-k).re
        cf = np.asarray(bank.coeffs)
        self._hermitian = bool(np.all(cf == np.conj(cf[:, :, ::-1, ::-1, ::-1])))

        self._forced = None
        if forced_velocity is not None:
            ix, iy = bank.index_of(forced_velocity)
            self._forced = (ix, iy)

        lib = _native.load()
        cparams, self._keep = _native.make_params(params)
        coeffs = np.ascontiguousarray(bank.coeffs_flat, dtype=np.complex64)
        retained = np.ascontiguousarray(bank.retained, dtype=np.int64)
        handle = ctypes.c_void_p()
        rc = lib.cw_create(
            ctypes.byref(cparams), self.width, self.height, self.device,
            _native.fptr(coeffs.view(np.float32)),
            retained.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), retained.size,
            int(_strip[0]), int(_strip[1]), ctypes.byref(handle),
        )
        _native.check(rc, None)
        self._h = handle
        self._idx_bytes = int(lib.cw_index_bytes(self._h))
        if self._forced is not None:
            _native.check(lib.cw_set_forced_velocity(self._h, *self._forced), self._h)
        if spectrum_backend == "naive":
            _native.check(lib.cw_set_backend(self._h, 1), self._h)
        self._device_timing = bool(device_timing)
        if self._device_timing:  # kernel milliseconds in last_timings (CUDA events)
            _native.check(lib.cw_set_timing(self._h, 1), self._h)
        self._detect = detect_threshold is not None
        self._max_det = int(max_detections)
        if self._detect:
            _native.check(lib.cw_set_detection(self._h, float(detect_threshold), self._max_det), self._h)

    # -- reference properties (pipeline.py:179-199) -------------------------

    @property
    def strategy(self) -> ExecStrategy:
        return self._strategy

    @property
    def latency(self) -> int:
        return self.params.mhat[2]

    @property
    def frames_seen(self) -> int:
        return int(_native.load().cw_frames_seen(self._h))

    @property
    def kernel_kind(self) -> str:
        """Which device path runs these parameters: "compiled" (a fused
        instance in the library), "jit" (the fused kernel compiled at run
        time for this geometry) or "runtime-geometry"."""
        return ("compiled", "jit", "runtime-geometry")[int(_native.load().cw_kernel_kind(self._h))]

    def set_strategy(self, strategy: ExecStrategy | str) -> None:
        """Accepted for compatibility; outputs are unaffected."""
        self._strategy = ExecStrategy.parse(strategy) if isinstance(strategy, str) else strategy

    # -- the hot entry ---------------------------------------------------------

    def process_frame(self, frame) -> WhitenedOutput | None:
        """Consume one frame; ``None`` until Mz frames were seen, then the
        whitened frame ``n - mhat_z`` (pipeline.py:201-294)."""
        frame = np.ascontiguousarray(frame, dtype=np.float32)
        if frame.shape != (self.height, self.width):
            raise ValueError(f"frame shape {frame.shape} != {(self.height, self.width)}")
        lib = _native.load()
        t0 = time.perf_counter()
        h, w = self.height, self.width
        res, pred, vidx = self._pool.take_outputs(h, w, self._idx_bytes)
        ready = ctypes.c_int32(0)
        fidx = ctypes.c_int64(-1)
        rc = lib.cw_push(self._h, frame.ctypes.data, res.ctypes.data, pred.ctypes.data, vidx.ctypes.data,
                         ctypes.byref(ready), ctypes.byref(fidx), None)
        _native.check(rc, self._h)
        self._set_timings(time.perf_counter() - t0, bool(ready.value))
        if not ready.value:
            return None
        out = self._wrap(int(fidx.value), res, pred, vidx, ticket=self.frames_seen - 1)
        if not self._hermitian:
            out.imag_peak = self._imag_peak_from_state(vidx)
        return out

    def _set_timings(self, seconds: float, ready: bool) -> None:
        """Reference keys (pipeline.py:210-285): warm-up frames report
        spectrum + pipeline, ready frames all five stages; the fused stages
        after the spectrum take no time of their own."""
        t = {"spectrum": seconds}
        if ready:
            t.update(conditioning=0.0, autocorr=0.0, filtering=0.0)
        t["pipeline"] = seconds
        if self._device_timing:
            ms, n = ctypes.c_double(), ctypes.c_int64()
            lib = _native.load()
            _native.check(lib.cw_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n)), self._h)
            t["kernel"] = ms.value / 1e3
        self.last_timings = t

    def _imag_peak_from_state(self, vidx) -> float:
        """max |Im sum_j c_j S_j| over the valid outputs (_kernels.py:338-341)
        for a non-Hermitian bank, from the spectrum of the frame just run."""
        p = self.params
        spec = self.spectrum()
        x0, x1, y0, y1 = valid_bounds(p, self.width, self.height)
        mhx, mhy, _ = p.mhat
        cy, cx = p.ky, p.kx
        band = spec[y0 + mhy:y1 + mhy + 1, x0 + mhx:x1 + mhx + 1, :,
                    cy - p.by:cy + p.by + 1, cx - p.bx:cx + p.bx + 1]
        v = vidx[y0 + mhy:y1 + mhy + 1, x0 + mhx:x1 + mhx + 1]
        coef = np.asarray(self.bank.coeffs, np.complex128)[v[..., 1], v[..., 0]]
        imag = np.abs(np.einsum("...k,...k->...", coef.reshape(coef.shape[:2] + (-1,)),
                                band.reshape(band.shape[:2] + (-1,))).imag)
        return float(imag.astype(np.float32).max()) if imag.size else 0.0

    def process_stream(self, frames, depth: int = 3, sample_format: str = "f32le",
                       scale: float = 1.0, offset: float = 0.0):
        """Pipelined ``process_frame`` over an iterable of (H, W) frames.

        Yields the same WhitenedOutput sequence as calling ``process_frame``
        on each frame (warm-up frames yield nothing), but keeps up to
        ``depth`` frames in flight so that the upload of frame n+1 and the
        download of frame n-1 overlap the kernel of frame n (cw_submit /
        cw_wait).  Pinned input frames (e.g. numpy views
        of ``torch.empty(..., pin_memory=True)``) give fully async uploads.

        ``sample_format="pgm16"`` takes frames as the raw big-endian uint16
        samples of a PGM16 sequence (dtype ">u2", e.g. from
        ``seqio.SequenceReader.read_raw``): they are uploaded as 16-bit words
        and de-quantised on the GPU as f32(f64(q) * scale + offset), the
        value ``seqio.read_sequence`` returns.
        """
        from collections import deque

        lib = _native.load()
        depth = max(1, min(int(depth), 6))
        h, w = self.height, self.width
        if sample_format not in ("f32le", "pgm16"):
            raise ValueError(f"unknown sample format {sample_format!r}")
        pgm = sample_format == "pgm16"
        if pgm and not scale > 0:
            raise ValueError("scale must be > 0")
        inflight: deque = deque()

        def collect(item):
            ticket, _frame, res, pred, vidx = item
            ready, fidx = ctypes.c_int32(0), ctypes.c_int64(-1)
            _native.check(lib.cw_wait(self._h, ticket, ctypes.byref(ready), ctypes.byref(fidx)), self._h)
            return self._wrap(int(fidx.value), res, pred, vidx, ticket=ticket) if ready.value else None

        try:
            for frame in frames:
                frame = np.ascontiguousarray(frame, dtype=">u2" if pgm else np.float32)
                if frame.shape != (h, w):
                    raise ValueError(f"frame shape {frame.shape} != {(h, w)}")
                res, pred, vidx = self._pool.take_outputs(h, w, self._idx_bytes)
                ticket = ctypes.c_int64(-1)
                rc = lib.cw_submit_raw(self._h, frame.ctypes.data, _native.FMT_PGM16 if pgm else _native.FMT_F32LE,
                                       float(scale), float(offset), res.ctypes.data, pred.ctypes.data,
                                       vidx.ctypes.data, ctypes.byref(ticket))
                _native.check(rc, self._h)
                inflight.append((ticket.value, frame, res, pred, vidx))
                while len(inflight) > depth:
                    out = collect(inflight.popleft())
                    if out is not None:
                        yield out
            while inflight:
                out = collect(inflight.popleft())
                if out is not None:
                    yield out
        finally:
            # the caller stopped early (break / close / GC) or a call failed:
            # wait for every outstanding frame before its pinned output block
            # (and input frame) can be recycled, so that no queued D2H copy
            # lands in a block a later call already owns
            while inflight:
                ticket = inflight.popleft()[0]
                if self._h:
                    lib.cw_wait(self._h, ticket, None, None)

    def process_resident(self, frames, depth: int = 3):
        """Pipelined ``process_frame`` over device-resident frames: an
        iterable of CUDA float32 (H, W) tensors on this pipeline's device,
        each complete when handed over (the producer is synchronised here)
        and left unchanged until its output is yielded.  Consecutive frame
        kernels are chained (cw_submit_resident): no frame
        copy, and a frame's kernel starts in the SM slots the previous one's
        early CTAs free.  Yields the WhitenedOutput of every ready frame, in
        order, with host arrays (downloaded while later frames run)."""
        import torch
        from collections import deque

        lib = _native.load()
        depth = max(1, min(int(depth), 6))
        h, w = self.height, self.width
        inflight: deque = deque()

        def collect(item):
            ticket, _frame, res, pred, vidx = item
            ready, fidx = ctypes.c_int32(0), ctypes.c_int64(-1)
            _native.check(lib.cw_wait(self._h, ticket, ctypes.byref(ready), ctypes.byref(fidx)), self._h)
            return self._wrap(int(fidx.value), res, pred, vidx, ticket=ticket) if ready.value else None

        try:
            for frame in frames:
                if (tuple(frame.shape) != (h, w) or frame.dtype != torch.float32 or not frame.is_cuda
                        or not frame.is_contiguous()):
                    raise ValueError(f"expected a contiguous CUDA float32 tensor of shape {(h, w)}")
                torch.cuda.current_stream(frame.device).synchronize()  # the frame is complete
                res, pred, vidx = self._pool.take_outputs(h, w, self._idx_bytes)
                ticket = ctypes.c_int64(-1)
                _native.check(lib.cw_submit_resident(self._h, ctypes.c_void_p(frame.data_ptr()), res.ctypes.data,
                                                     pred.ctypes.data, vidx.ctypes.data, ctypes.byref(ticket)),
                              self._h)
                inflight.append((ticket.value, frame, res, pred, vidx))
                while len(inflight) > depth:
                    out = collect(inflight.popleft())
                    if out is not None:
                        yield out
            while inflight:
                out = collect(inflight.popleft())
                if out is not None:
                    yield out
        finally:
            while inflight:
                ticket = inflight.popleft()[0]
                if self._h:
                    lib.cw_wait(self._h, ticket, None, None)

    def process_frame_device(self, frame) -> WhitenedOutput | None:
        """``process_frame`` for a frame already in device memory: a CUDA
        float32 (H, W) torch tensor on this pipeline's device (e.g. a strip
        assembled from NCCL halo receives).  Runs on torch's current
        stream; outputs are copied to fresh host arrays."""
        import torch

        if tuple(frame.shape) != (self.height, self.width) or frame.dtype != torch.float32 or not frame.is_cuda:
            raise ValueError(f"expected a CUDA float32 tensor of shape {(self.height, self.width)}")
        frame = frame.contiguous()
        lib = _native.load()
        t0 = time.perf_counter()
        ready = ctypes.c_int32(0)
        fidx = ctypes.c_int64(-1)
        # run on a dedicated stream ordered after the producer of `frame`
        # (handle 0 at the C ABI would mean the pipeline's own stream)
        if getattr(self, "_tstream", None) is None:
            self._tstream = torch.cuda.Stream(device=frame.device)
        stream = self._tstream
        stream.wait_stream(torch.cuda.current_stream(frame.device))
        frame.record_stream(stream)
        rc = lib.cw_push_device(self._h, ctypes.c_void_p(frame.data_ptr()), ctypes.byref(ready),
                                ctypes.byref(fidx), ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc, self._h)
        stream.synchronize()
        if not ready.value:
            self._set_timings(time.perf_counter() - t0, False)
            return None
        res_p, pred_p, vidx_p = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(lib.cw_device_outputs(self._h, ctypes.byref(res_p), ctypes.byref(pred_p),
                                            ctypes.byref(vidx_p)), self._h)
        h, w = self.height, self.width
        res = np.empty((h, w), np.float32)
        pred = np.empty((h, w), np.float32)
        vidx = np.empty((h, w, 2), np.uint8 if self._idx_bytes == 1 else np.uint16)
        for dst, src in ((res, res_p), (pred, pred_p), (vidx, vidx_p)):
            _native.check(lib.cw_copy_to_host(self._h, dst.ctypes.data, src, dst.nbytes), self._h)
        self._set_timings(time.perf_counter() - t0, True)
        out = self._wrap(int(fidx.value), res, pred, vidx, ticket=self.frames_seen - 1)
        if not self._hermitian:
            out.imag_peak = self._imag_peak_from_state(vidx)
        return out

    def _indices_of(self, vidx) -> np.ndarray:
        """(H, W, 2) int32 [ix, iy] from the device's index pairs."""
        if self._idx_bytes == 1:
            return self._lut_i[vidx.view(np.uint16).reshape(vidx.shape[:2])]
        return vidx.astype(np.int32)

    def _velocities_of(self, vidx, dtype=np.float64) -> np.ndarray:
        """(H, W, 2) [vx, vy] lags of the device's index pairs (float64 as
        flow.VelocityField; ``dtype`` float32 for velocity files)."""
        if self._idx_bytes == 1:
            lut = self._lut_v if dtype == np.float64 else self._lut_v.astype(dtype)
            return np.take(lut, vidx.view(np.uint16).reshape(vidx.shape[:2]), axis=0)
        return np.stack([self._lag_x[vidx[..., 0]], self._lag_y[vidx[..., 1]]], axis=-1).astype(dtype)

    def _wrap(self, frame_index, res, pred, vidx, ticket=None) -> WhitenedOutput:
        out = WhitenedOutput(frame_index=frame_index, residual=res, prediction=pred,
                             velocity=_LazyVelocityField(vidx, self),
                             mask=self.mask, imag_peak=0.0 if self._hermitian else float("nan"))
        if self._detect and ticket is not None:
            out.detections, out.metrics = self._fetch_detections(ticket)
        return out

    def _fetch_detections(self, ticket):
        lib = _native.load()
        n = ctypes.c_int32(0)
        buf = np.empty((self._max_det, 3), np.float32)
        st = np.zeros(5, np.float64)
        _native.check(lib.cw_detections(self._h, int(ticket), ctypes.byref(n), _native.fptr(buf), self._max_det,
                                        st.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), self._h)
        k = min(n.value, self._max_det)
        det = buf[:k].astype(np.float64)
        det = det[np.lexsort((det[:, 0], det[:, 1]))] if k else det
        nval = int(st[4])
        metrics = {
            "peak_abs_residual": float(st[0]), "peak_x": int(st[1]), "peak_y": int(st[2]),
            "residual_rms": float(np.sqrt(st[3] / nval)) if nval else 0.0,
            "n_valid": nval, "n_detections": int(n.value), "truncated": n.value > self._max_det,
        }
        return det, metrics

    # -- checkpoint / resume -----------------------------------------------

    def snapshot(self) -> np.ndarray:
        """The whole stream state (observer + smoothing state, frame ring,
        counters) as a uint8 array; ``restore`` continues from it."""
        lib = _native.load()
        n = ctypes.c_size_t(0)
        _native.check(lib.cw_snapshot_size(self._h, ctypes.byref(n)), self._h)
        buf = np.empty(n.value, np.uint8)
        _native.check(lib.cw_snapshot(self._h, buf.ctypes.data, buf.nbytes), self._h)
        return buf

    def restore(self, snap) -> None:
        """Resume from ``snapshot()`` of a pipeline with the same geometry."""
        snap = np.ascontiguousarray(snap, dtype=np.uint8)
        _native.check(_native.load().cw_restore(self._h, snap.ctypes.data, snap.nbytes), self._h)

    # -- parity views (tests) ------------------------------------------------

    def spectrum(self) -> np.ndarray:
        """S of the last frame as (H, W, Mz, My, Mx) complex128 (reference
        SpectrumField.bins layout), rebuilt from the observer state."""
        p = self.params
        out = np.zeros((self.height, self.width, p.mz, p.my, p.mx), np.complex128)
        rc = _native.load().cw_read_view(self._h, 0, out.ctypes.data, out.nbytes)
        _native.check(rc, self._h)
        return out

    def smoothed_state(self) -> np.ndarray:
        """T^ (H, W, My, Mx) complex128: the kz-collapsed smoothed power whose
        lag transform is the reference R^ (flow.py:87-114)."""
        p = self.params
        out = np.zeros((self.height, self.width, p.my, p.mx), np.complex128)
        rc = _native.load().cw_read_view(self._h, 1, out.ctypes.data, out.nbytes)
        _native.check(rc, self._h)
        return out

    def launch_info(self) -> dict:
        k, g, b, s = (ctypes.c_int32() for _ in range(4))
        _native.check(_native.load().cw_launch_info(self._h, *(ctypes.byref(v) for v in (k, g, b, s))), self._h)
        return {"kernels_per_push": k.value, "grid": g.value, "block": b.value, "smem_bytes": s.value}

    # -- lifetime ---------------------------------------------------------------

    def close(self) -> None:
        if getattr(self, "_h", None):
            _native.load().cw_destroy(self._h)
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


def rhat_from_state(that: np.ndarray, params: FilterParams) -> np.ndarray:
    """R^(ly, lx) = Re sum_k e^{-j2pi(kx lx/Mx + ky ly/My)} T^(ky, kx): the
    reference's smoothed autocorrelation recovered from T^ (flow.py:100-114,
    _kernels.py:230-258 with the kz collapse already applied)."""
    kx = np.arange(params.mx) - params.kx
    ky = np.arange(params.my) - params.ky
    axl = np.exp(-2j * np.pi * np.outer(np.asarray(params.lag_grid_x), kx) / params.mx)
    ayl = np.exp(-2j * np.pi * np.outer(np.asarray(params.lag_grid_y), ky) / params.my)
    return np.einsum("lx,my,...yx->...ml", axl, ayl, that).real
