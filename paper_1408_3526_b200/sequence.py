"""Whitening a stored sequence end to end: ingest -> GPU -> egress (§8f rank 1).

``filter_sequence(input_dir, out_dir, params)`` produces the same files as
the reference's ``clutterwhiten filter`` (cli._cmd_filter, cli.py:230-306):

* ``out_dir/``            residual sequence (header meta: source, input,
                          first_frame_index, latency_frames)
* ``out_dir/prediction/`` prediction sequence (``emit_prediction``)
* ``out_dir/velocity.f32`` + ``velocity.json`` (vx, vy) f32 per pixel
                          (``emit_velocity``; sidecar of cli.py:211-227)
* ``metrics`` CSV          METRICS_HEADER rows (cli.py:36-39, 157-208)
* ``out_dir/run_meta.json`` the run record (cli.py:59-64, 291-305)

but streams instead of holding the sequence in memory, and keeps the GPU
fed: a reader thread pulls each frame's raw payload bytes straight into a
pinned staging buffer (no host-side conversion: float32 frames upload as
is, PGM16 frames upload as 16-bit words and are decoded on the GPU by
``cw_submit_raw``), the main thread keeps ``depth`` frames in flight
(upload / fused kernel / download on three CUDA streams), and a writer
thread appends the outputs to disk.

Metrics: without ground truth the row comes from the fused threshold
epilogue in the frame kernel (peak |res| with the reference's first-in-
row-major tie rule, and sum of f64 squares over the valid region ->
background RMS); with ``ground_truth.json`` next to the input (written by
the reference's ``simulate``) the target-disk exclusion, hit flag and
velocity errors are computed on the host exactly as cli.compute_metrics_row.
"""

from __future__ import annotations

import ctypes
import json
import math
import queue
import threading
import time
from dataclasses import dataclass
from pathlib import Path
from types import SimpleNamespace

import numpy as np

from . import __version__, _native
from .params import FilterParams, default_params, params_as_dict
from .pipeline import Pipeline, valid_bounds
from .seqio import SequenceError, SequenceReader, SequenceWriter

__all__ = ["METRICS_HEADER", "MetricsRow", "GroundTruthLite", "load_ground_truth", "target_exclusion_radius",
           "metrics_row", "filter_sequence", "flow_sequence"]

GROUND_TRUTH_NAME = "ground_truth.json"
RUN_META_NAME = "run_meta.json"
METRICS_HEADER = (
    "frame_index,background_rms,peak_abs_residual,peak_x,peak_y,"
    "target_x,target_y,hit,vel_err_median,vel_err_within_quarter"
)


@dataclass
class MetricsRow:
    """One metrics CSV row (cli.py:114-139)."""

    frame_index: int
    background_rms: float
    peak_abs_residual: float
    peak_x: int
    peak_y: int
    target_x: float | None = None
    target_y: float | None = None
    hit: bool | None = None
    vel_err_median: float | None = None
    vel_err_within_quarter: float | None = None

    def csv(self) -> str:
        def fmt(v):
            return "" if v is None else format(v, ".6g")

        hit = "" if self.hit is None else str(int(self.hit))
        return (f"{self.frame_index},{self.background_rms:.6g},{self.peak_abs_residual:.6g},"
                f"{self.peak_x},{self.peak_y},{fmt(self.target_x)},{fmt(self.target_y)},{hit},"
                f"{fmt(self.vel_err_median)},{fmt(self.vel_err_within_quarter)}")


@dataclass
class GroundTruthLite:
    """The fields of the reference's ground_truth.json the metrics use
    (scenegen.GroundTruth.to_json_dict, scenegen.py:73-85)."""

    clutter_velocity: tuple[float, float]
    target_centers: np.ndarray | None
    psf_sigma: float
    target_peak: float | None
    target_truncation: float


def load_ground_truth(seq_dir) -> GroundTruthLite | None:
    path = Path(seq_dir) / GROUND_TRUTH_NAME
    if not path.is_file():
        return None
    data = json.loads(path.read_text(encoding="utf-8"))
    cfg = data["config"]
    centers = data.get("target_centers")
    return GroundTruthLite(
        clutter_velocity=tuple(float(v) for v in data["clutter_velocity"]),
        target_centers=None if centers is None else np.asarray(centers, dtype=np.float64),
        psf_sigma=float(cfg["psf_sigma"]),
        target_peak=None if cfg.get("target_peak") is None else float(cfg["target_peak"]),
        target_truncation=float(cfg["target_truncation"]),
    )


def target_exclusion_radius(params: FilterParams, truth: GroundTruthLite) -> int:
    """Truncation-disk radius plus the analysis-window reach (cli.py:145-154)."""
    radius = truth.psf_sigma * math.sqrt(
        2.0 * math.log(max(truth.target_peak or 1.0, truth.target_truncation * 2) / truth.target_truncation))
    return int(math.ceil(radius)) + max(params.kx, params.ky) + 1


def metrics_row(out, params: FilterParams, truth: GroundTruthLite | None) -> MetricsRow:
    """cli.compute_metrics_row (cli.py:157-208).  Without ground truth and
    with the fused epilogue's stats on ``out.metrics`` no host pass over the
    residual is needed."""
    m = getattr(out, "metrics", None)
    if truth is None and m is not None:
        rms = math.sqrt(m["sum_sq"] / m["n_valid"]) if m["n_valid"] else 0.0
        return MetricsRow(out.frame_index, rms, m["peak_abs_residual"], m["peak_x"], m["peak_y"])
    res, mask = out.residual, out.mask
    absres = np.abs(res)
    flat = int(np.argmax(np.where(mask, absres, -1.0)))
    py, px = np.unravel_index(flat, res.shape)
    row = MetricsRow(out.frame_index, 0.0, float(absres[py, px]), int(px), int(py))
    bg_mask = mask.copy()
    if truth is not None and truth.target_centers is not None:
        cx, cy = truth.target_centers[out.frame_index]
        row.target_x, row.target_y = float(cx), float(cy)
        row.hit = bool(max(abs(px - cx), abs(py - cy)) <= 1.0)
        excl = target_exclusion_radius(params, truth)
        ys = np.arange(res.shape[0])[:, None]
        xs = np.arange(res.shape[1])[None, :]
        bg_mask &= np.maximum(np.abs(xs - cx), np.abs(ys - cy)) > excl
    bg = res[bg_mask]
    row.background_rms = float(np.sqrt(np.mean(bg.astype(np.float64) ** 2))) if bg.size else 0.0
    if truth is not None:
        cvx, cvy = truth.clutter_velocity
        vel = out.velocity.velocities
        err = np.maximum(np.abs(vel[..., 0] - cvx), np.abs(vel[..., 1] - cvy))
        err = err[params.my - 1:, params.mx - 1:].ravel()
        row.vel_err_median = float(np.median(err))
        row.vel_err_within_quarter = float(np.mean(err <= 0.25))
    return row


class _Out:
    """Minimal WhitenedOutput view handed to metrics_row on the writer thread."""

    def __init__(self, frame_index, residual, mask, velocity, metrics):
        self.frame_index, self.residual, self.mask = frame_index, residual, mask
        self.velocity, self.metrics = velocity, metrics


def _pinned(nbytes: int) -> np.ndarray:
    import torch

    return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy()


def _stream(reader: SequenceReader, pipe: Pipeline, consume, *, want_pred: bool, want_stats: bool,
            depth: int) -> float:
    """Run every frame of ``reader`` through ``pipe``: a reader thread fills
    pinned payload buffers, the calling thread keeps ``depth`` frames in
    flight through cw_submit_raw / cw_wait, and a writer thread calls
    ``consume(frame_index, input_index, residual, prediction, vidx, stats)``
    for each ready output in order (its arrays are recycled afterwards).
    Returns the wall-clock seconds of the run."""
    lib = _native.load()
    h, w = reader.shape
    hdr = reader.header
    depth = max(1, min(int(depth), 6))
    n_in, n_out = depth + 3, depth + 4
    free_in: queue.Queue = queue.Queue()
    for _ in range(n_in):
        free_in.put(_pinned(reader.frame_bytes))
    free_out: queue.Queue = queue.Queue()
    for _ in range(n_out):
        free_out.put((_pinned(h * w * 4).view(np.float32).reshape(h, w),
                      _pinned(h * w * 4).view(np.float32).reshape(h, w),
                      _pinned(h * w * 2 * pipe._idx_bytes).view(np.uint8 if pipe._idx_bytes == 1 else np.uint16)
                      .reshape(h, w, 2)))
    ready_in: queue.Queue = queue.Queue(maxsize=n_in)
    to_write: queue.Queue = queue.Queue(maxsize=n_out)
    errors: list[BaseException] = []

    def read_loop():
        try:
            for t in range(len(reader)):
                buf = free_in.get()
                if buf is None:
                    return
                reader.read_raw(t, buf)
                ready_in.put((t, buf))
        except BaseException as exc:  # surfaced on the calling thread
            errors.append(exc)
        ready_in.put(None)

    def write_loop():
        # After a failed consume() the loop keeps draining to_write (without
        # consuming) so that every output set goes back to free_out and the
        # calling thread, blocked in free_out.get() or to_write.put(), wakes
        # up, sees `errors` and stops submitting.
        failed = False
        while True:
            item = to_write.get()
            if item is None:
                return
            fidx, t_in, outs, stats = item
            if not failed:
                try:
                    consume(fidx, t_in, outs[0], outs[1], outs[2], stats)
                except BaseException as exc:
                    errors.append(exc)
                    failed = True
            free_out.put(outs)

    inflight = []

    def collect():
        ticket, buf, outs = inflight.pop(0)
        ready, fidx = ctypes.c_int32(0), ctypes.c_int64(-1)
        _native.check(lib.cw_wait(pipe._h, ticket, ctypes.byref(ready), ctypes.byref(fidx)), pipe._h)
        free_in.put(buf)
        if not ready.value:
            free_out.put(outs)
            return
        stats = None
        if want_stats:
            st = np.zeros(5, np.float64)
            n = ctypes.c_int32(0)
            _native.check(lib.cw_detections(pipe._h, ticket, ctypes.byref(n), None, 0,
                                            st.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), pipe._h)
            stats = {"peak_abs_residual": float(st[0]), "peak_x": int(st[1]), "peak_y": int(st[2]),
                     "sum_sq": float(st[3]), "n_valid": int(st[4])}
        to_write.put((int(fidx.value), ticket, outs, stats))

    reader_t = threading.Thread(target=read_loop, name="cw-ingest", daemon=True)
    writer_t = threading.Thread(target=write_loop, name="cw-egress", daemon=True)
    fmt = _native.FMT_PGM16 if reader.pgm else _native.FMT_F32LE
    t0 = time.perf_counter()
    reader_t.start()
    writer_t.start()
    try:
        while not errors:
            item = ready_in.get()
            if item is None:
                break
            _, buf = item
            res, pred, vidx = free_out.get()
            ticket = ctypes.c_int64(-1)
            _native.check(lib.cw_submit_raw(
                pipe._h, ctypes.c_void_p(buf.ctypes.data), fmt, float(hdr.scale), float(hdr.offset),
                _native.fptr(res), _native.fptr(pred) if want_pred else None,
                vidx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), ctypes.byref(ticket)), pipe._h)
            inflight.append((ticket.value, buf, (res, pred, vidx)))
            while len(inflight) > depth:
                collect()
        while inflight and not errors:
            collect()
    finally:
        # never leave a DMA in flight into buffers this function drops
        for ticket, _buf, _outs in inflight:
            lib.cw_wait(pipe._h, ticket, None, None)
        inflight.clear()
        free_in.put(None)  # unblock the reader if it waits for a buffer
        to_write.put(None)
        writer_t.join()
        reader_t.join(timeout=5.0)
    if errors:
        raise errors[0]
    return time.perf_counter() - t0


def filter_sequence(input_dir, out_dir, params: FilterParams | None = None, *, dtype: str = "f32le",
                    emit_prediction: bool = False, emit_velocity: bool = False, metrics=None,
                    spectrum_backend: str = "recursive", depth: int = 3, device: int = 0) -> dict:
    """Whiten the sequence in ``input_dir`` into ``out_dir`` (cli._cmd_filter
    semantics, cli.py:230-306); returns the run-meta dict it also writes."""
    params = default_params() if params is None else params
    out_dir = Path(out_dir)
    truth = load_ground_truth(input_dir)
    want_metrics = metrics is not None
    with SequenceReader(input_dir) as reader:
        h, w = reader.shape
        hdr = reader.header
        out_dir.mkdir(parents=True, exist_ok=True)
        res_w = SequenceWriter(out_dir, w, h, dtype=dtype)
        pred_w = SequenceWriter(out_dir / "prediction", w, h, dtype=dtype) if emit_prediction else None
        vel_fh = open(out_dir / "velocity.f32", "wb") if emit_velocity else None
        rows: list[MetricsRow] = []
        first_index = [None]
        with Pipeline(params, w, h, spectrum_backend=spectrum_backend, device=device,
                      detect_threshold=0.0 if want_metrics else None, max_detections=0) as pipe:

            def consume(fidx, _t, res, pred, vidx, stats):
                if first_index[0] is None:
                    first_index[0] = fidx
                res_w.append(res)
                if pred_w is not None:
                    pred_w.append(pred)
                if vel_fh is not None:  # f64 lags rounded to f32
                    vel_fh.write(pipe._velocities_of(vidx, np.dtype("<f4")).data)
                if want_metrics:
                    # metrics from the float64 lags, as cli.compute_metrics_row
                    velocity = (None if truth is None
                                else SimpleNamespace(velocities=pipe._velocities_of(vidx)))
                    rows.append(metrics_row(_Out(fidx, res, pipe.mask, velocity, stats), params, truth))

            try:
                elapsed = _stream(reader, pipe, consume, want_pred=pred_w is not None, want_stats=want_metrics,
                                  depth=depth)
            finally:
                if vel_fh is not None:
                    vel_fh.close()
            bank_seconds = pipe.bank.build_seconds
    n_out = res_w.count
    if n_out == 0:
        raise SequenceError("sequence shorter than the temporal window")
    seq_meta = {"source": "filter", "input": str(input_dir), "first_frame_index": first_index[0],
                "latency_frames": params.latency}
    res_w.meta = dict(seq_meta)
    res_w.close()
    if pred_w is not None:
        pred_w.meta = dict(seq_meta, source="filter-prediction")
        pred_w.close()
    if emit_velocity:
        _velocity_sidecar(out_dir, n_out, w, h, first_index[0])
    if want_metrics:
        with open(metrics, "w", encoding="utf-8") as fh:
            fh.write(METRICS_HEADER + "\n")
            for row in rows:
                fh.write(row.csv() + "\n")
    ox_lo, ox_hi, oy_lo, oy_hi = valid_bounds(params, w, h)
    return _run_meta(out_dir, {
        "command": "filter", "params": params_as_dict(params), "strategy": "serial",
        "backend": spectrum_backend, "input": str(input_dir), "input_seed": hdr.meta.get("seed"),
        "frames_in": len(reader), "frames_out": n_out,
        "valid_region": {"x": [ox_lo, ox_hi], "y": [oy_lo, oy_hi]},
        "latency_frames": params.latency, "bank_build_seconds": bank_seconds, "seconds": elapsed,
        "device": "cuda", "sample_format": hdr.dtype,
    })


def flow_sequence(input_dir, out_dir, params: FilterParams | None = None, *, fmt: str = "f32",
                  depth: int = 3, device: int = 0) -> dict:
    """Per-frame velocity fields of the sequence in ``input_dir``
    (cli._cmd_flow, cli.py:312-357): ``velocity.f32`` + ``velocity.json``
    (fmt "f32") or ``velocity.csv`` rows "frame,y,x,vx,vy" over the anchor
    region (fmt "csv"); frames are numbered by input index."""
    if fmt not in ("f32", "csv"):
        raise ValueError(f"unknown flow format {fmt!r}")
    params = default_params() if params is None else params
    out_dir = Path(out_dir)
    with SequenceReader(input_dir) as reader:
        h, w = reader.shape
        hdr = reader.header
        out_dir.mkdir(parents=True, exist_ok=True)
        fh = open(out_dir / ("velocity.f32" if fmt == "f32" else "velocity.csv"), "w" + ("b" if fmt == "f32" else ""),
                  **({} if fmt == "f32" else {"encoding": "utf-8"}))
        if fmt == "csv":
            fh.write("frame,y,x,vx,vy\n")
        first, count = [None], [0]
        ys, xs = np.mgrid[params.my - 1:h, params.mx - 1:w]
        with Pipeline(params, w, h, device=device) as pipe:
            def consume(_fidx, t_in, _res, _pred, vidx, _stats):
                vel = pipe._velocities_of(vidx, np.dtype("<f4"))
                if first[0] is None:
                    first[0] = t_in
                count[0] += 1
                if fmt == "f32":
                    fh.write(vel.data)
                else:
                    va = vel[params.my - 1:, params.mx - 1:]
                    fh.write("".join(f"{t_in},{y},{x},{vx:.6g},{vy:.6g}\n" for y, x, vx, vy in
                                     zip(ys.ravel().tolist(), xs.ravel().tolist(),
                                         va[..., 0].ravel().tolist(), va[..., 1].ravel().tolist())))

            try:
                _stream(reader, pipe, consume, want_pred=False, want_stats=False, depth=depth)
            finally:
                fh.close()
    if count[0] == 0:
        raise SequenceError("sequence shorter than the temporal window")
    if fmt == "f32":
        _velocity_sidecar(out_dir, count[0], w, h, first[0])
    return _run_meta(out_dir, {
        "command": "flow", "params": params_as_dict(params), "strategy": "serial", "input": str(input_dir),
        "input_seed": hdr.meta.get("seed"), "frames_in": len(reader), "fields_out": count[0], "device": "cuda",
    })


def _velocity_sidecar(out_dir: Path, count: int, width: int, height: int, first_index) -> None:
    """velocity.json next to velocity.f32 (cli.py:211-227)."""
    with open(out_dir / "velocity.json", "w", encoding="utf-8") as fh:
        json.dump({"width": width, "height": height, "frame_count": count, "channels": 2,
                   "components": ["vx", "vy"], "dtype": "f32le", "first_frame_index": first_index}, fh, indent=2)
        fh.write("\n")


def _run_meta(out_dir: Path, payload: dict) -> dict:
    """run_meta.json (cli.py:59-64)."""
    payload = dict(payload, version=__version__)
    with open(out_dir / RUN_META_NAME, "w", encoding="utf-8") as fh:
        json.dump(payload, fh, indent=2, default=float)
        fh.write("\n")
    return payload
