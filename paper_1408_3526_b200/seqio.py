"""Image-sequence storage compatible with the reference's seqio (§8f rank 1).

On-disk formats are those of /root/reference/pkg/src/clutterwhiten/seqio.py
(restated, not imported): a directory with ``header.json`` and either one
``frames.f32`` payload (little-endian float32, frames in C order) or one
``frame_NNNNNN.pgm`` per frame (binary P5, maxval 65535, big-endian samples
quantised as q = rint((v - offset) / scale)).  Error type and messages match
(``SequenceError``, seqio.py:29-30, 131-204), so callers' ``except`` clauses
and tests carry over.

Beyond the reference's whole-sequence ``read_sequence`` / ``write_sequence``
(which hold every frame in host memory) this module streams:

* ``SequenceReader`` hands out one frame's RAW payload bytes at a time
  (``read_raw(t, out)``: a ``readinto`` straight into a caller buffer, e.g.
  a pinned staging buffer) — float32 frames need no conversion on the host
  and PGM16 frames are byte-swapped and de-quantised on the GPU
  (``cw_submit_raw``), so the host only moves bytes.
* ``SequenceWriter`` appends f32le frames as they arrive and writes the
  header on ``close()``; pgm16 output keeps the reference's global-range
  quantisation (scale/offset from the min/max of ALL frames,
  seqio.py:98-105), so it buffers frames until ``close()``.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

__all__ = [
    "SequenceError", "SequenceHeader", "read_sequence", "write_sequence",
    "read_header", "SequenceReader", "SequenceWriter", "HEADER_NAME", "RAW_NAME", "DTYPES",
]

HEADER_NAME = "header.json"
RAW_NAME = "frames.f32"
DTYPES = ("f32le", "pgm16")


class SequenceError(Exception):
    """Malformed, truncated or inconsistent sequence storage (seqio.py:29-30)."""


@dataclass
class SequenceHeader:
    """Sequence geometry and quantisation (seqio.py:33-78)."""

    width: int
    height: int
    frame_count: int
    dtype: str = "f32le"
    scale: float = 1.0
    offset: float = 0.0
    meta: dict = field(default_factory=dict)

    def validate(self) -> None:
        if self.dtype not in DTYPES:
            raise SequenceError(f"unknown sequence dtype {self.dtype!r}")
        if self.width < 1 or self.height < 1 or self.frame_count < 0:
            raise SequenceError("non-positive sequence geometry")
        if self.scale <= 0:
            raise SequenceError(f"scale must be > 0, got {self.scale}")

    def to_json_dict(self) -> dict:
        return {"width": self.width, "height": self.height, "frame_count": self.frame_count,
                "dtype": self.dtype, "scale": self.scale, "offset": self.offset, "meta": self.meta}

    @classmethod
    def from_json_dict(cls, data: dict) -> "SequenceHeader":
        try:
            hdr = cls(width=int(data["width"]), height=int(data["height"]),
                      frame_count=int(data["frame_count"]), dtype=str(data.get("dtype", "f32le")),
                      scale=float(data.get("scale", 1.0)), offset=float(data.get("offset", 0.0)),
                      meta=dict(data.get("meta", {})))
        except (KeyError, TypeError, ValueError) as exc:
            raise SequenceError(f"malformed sequence header: {exc}") from exc
        hdr.validate()
        return hdr


def pgm_name(t: int) -> str:
    return f"frame_{t:06d}.pgm"


def _write_header(path: Path, header: SequenceHeader) -> None:
    with open(path / HEADER_NAME, "w", encoding="utf-8") as fh:
        json.dump(header.to_json_dict(), fh, indent=2)
        fh.write("\n")


def read_header(path) -> SequenceHeader:
    path = Path(path)
    hp = path / HEADER_NAME
    if not hp.is_file():
        raise SequenceError(f"missing {HEADER_NAME} in {path}")
    try:
        with open(hp, "r", encoding="utf-8") as fh:
            return SequenceHeader.from_json_dict(json.load(fh))
    except json.JSONDecodeError as exc:
        raise SequenceError(f"malformed sequence header: {exc}") from exc


def _pgm_range(frames: np.ndarray, scale, offset):
    """Default quantisation: the data range over all frames (seqio.py:98-105)."""
    lo = float(frames.min()) if frames.size else 0.0
    hi = float(frames.max()) if frames.size else 1.0
    if offset is None:
        offset = lo
    if scale is None:
        span = hi - offset
        scale = span / 65535.0 if span > 0 else 1.0
    return float(scale), float(offset)


def _pgm_bytes(frame: np.ndarray, scale: float, offset: float) -> bytes:
    h, w = frame.shape
    q = np.clip(np.rint((frame.astype(np.float64) - offset) / scale), 0, 65535).astype(">u2")
    return f"P5\n{w} {h}\n65535\n".encode("ascii") + q.tobytes()


def write_sequence(frames, path, dtype: str = "f32le", meta: dict | None = None,
                   scale: float | None = None, offset: float | None = None) -> SequenceHeader:
    """Write (T, H, W) frames as a sequence directory (seqio.py:80-128)."""
    frames = np.asarray(frames, dtype=np.float32)
    if frames.ndim != 3:
        raise SequenceError(f"expected (T, H, W) frames, got shape {frames.shape}")
    if dtype not in DTYPES:
        raise SequenceError(f"unknown sequence dtype {dtype!r}")
    t, h, w = frames.shape
    path = Path(path)
    path.mkdir(parents=True, exist_ok=True)
    if dtype == "pgm16":
        scale, offset = _pgm_range(frames, scale, offset)
    else:
        scale = 1.0 if scale is None else scale
        offset = 0.0 if offset is None else offset
    header = SequenceHeader(w, h, t, dtype, float(scale), float(offset), dict(meta or {}))
    header.validate()
    if dtype == "f32le":
        with open(path / RAW_NAME, "wb") as fh:
            fh.write(frames.astype("<f4", copy=False).tobytes())
    else:
        for i in range(t):
            with open(path / pgm_name(i), "wb") as fh:
                fh.write(_pgm_bytes(frames[i], header.scale, header.offset))
    _write_header(path, header)
    return header


_WS = frozenset(b" \t\n\r\x0b\x0c")  # bytes.isspace()


def _pgm_payload_offset(data: bytes, name: str, width: int, height: int) -> int:
    """Parse "P5 <w> <h> <maxval>" (comments and any whitespace allowed,
    one whitespace byte after maxval; seqio.py:131-169); returns the byte
    offset of the sample payload after checking geometry and length."""
    tokens: list[bytes] = []
    pos, n = 0, len(data)
    while len(tokens) < 4:
        if pos >= n:
            raise SequenceError(f"{name}: truncated PGM header")
        c = data[pos]
        if c == 0x23:  # '#': comment to end of line
            nl = data.find(b"\n", pos)
            pos = n if nl < 0 else nl + 1
        elif c in _WS:
            pos += 1
        else:
            end = pos
            while end < n and data[end] not in _WS:
                end += 1
            tokens.append(data[pos:end])
            pos = end
    pos += 1
    if tokens[0] != b"P5":
        raise SequenceError(f"{name}: not a binary PGM (P5)")
    try:
        pw, ph, maxval = (int(t) for t in tokens[1:4])
    except ValueError as exc:
        raise SequenceError(f"{name}: malformed PGM header") from exc
    if (pw, ph) != (width, height):
        raise SequenceError(f"{name}: frame is {pw}x{ph}, header says {width}x{height}")
    if maxval != 65535:
        raise SequenceError(f"{name}: expected 16-bit PGM, maxval {maxval}")
    if n - pos < width * height * 2:
        raise SequenceError(f"{name}: truncated PGM payload")
    return pos


class SequenceReader:
    """Frame-at-a-time access to a sequence directory.

    ``raw_dtype`` is the payload sample type ("<f4" or ">u2");
    ``read_raw(t, out)`` fills ``out`` (any writable buffer of
    ``frame_bytes`` bytes, e.g. a pinned numpy view) with frame t's payload;
    ``read(t)`` returns the de-quantised float32 frame exactly as
    ``read_sequence`` does (f32(f64(q) * scale + offset) for pgm16).
    """

    def __init__(self, path):
        self.path = Path(path)
        self.header = read_header(self.path)
        h = self.header
        self.pgm = h.dtype == "pgm16"
        self.raw_dtype = ">u2" if self.pgm else "<f4"
        self.frame_bytes = h.width * h.height * (2 if self.pgm else 4)
        self._fh = None
        if not self.pgm:
            raw = self.path / RAW_NAME
            if not raw.is_file():
                raise SequenceError(f"missing {RAW_NAME} in {self.path}")
            have = raw.stat().st_size // 4
            want = h.frame_count * h.height * h.width
            if have != want or raw.stat().st_size % 4:
                raise SequenceError(f"{RAW_NAME} holds {have} values, expected {want}")
            self._fh = open(raw, "rb", buffering=0)

    def __len__(self) -> int:
        return self.header.frame_count

    @property
    def shape(self) -> tuple[int, int]:
        return self.header.height, self.header.width

    def read_raw(self, t: int, out) -> None:
        if not 0 <= t < self.header.frame_count:
            raise IndexError(t)
        mv = memoryview(out).cast("B")
        if len(mv) < self.frame_bytes:
            raise ValueError("output buffer smaller than one frame")
        mv = mv[: self.frame_bytes]
        if not self.pgm:
            got = os.preadv(self._fh.fileno(), [mv], t * self.frame_bytes)
            if got != self.frame_bytes:
                raise SequenceError(f"{RAW_NAME}: short read at frame {t}")
            return
        name = pgm_name(t)
        p = self.path / name
        try:
            data = p.read_bytes()
        except FileNotFoundError as exc:
            raise SequenceError(f"missing {name} in {self.path}") from exc
        pos = _pgm_payload_offset(data, name, self.header.width, self.header.height)
        mv[:] = data[pos: pos + self.frame_bytes]

    def read(self, t: int) -> np.ndarray:
        h, w = self.shape
        raw = np.empty((h, w), dtype=self.raw_dtype)
        self.read_raw(t, raw)
        if not self.pgm:
            return raw.astype(np.float32)
        return (raw.astype(np.float64) * self.header.scale + self.header.offset).astype(np.float32)

    def close(self) -> None:
        if self._fh is not None:
            self._fh.close()
            self._fh = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def read_sequence(path):
    """(frames (T, H, W) float32, header) (seqio.py:172-204)."""
    with SequenceReader(path) as rd:
        h, w = rd.shape
        frames = np.empty((len(rd), h, w), dtype=np.float32)
        for t in range(len(rd)):
            frames[t] = rd.read(t)
        return frames, rd.header


class SequenceWriter:
    """Streaming sequence writer: ``append(frame)`` per (H, W) float32 frame,
    ``close()`` writes header.json (and, for pgm16, the quantised frames)."""

    def __init__(self, path, width: int, height: int, dtype: str = "f32le", meta: dict | None = None):
        if dtype not in DTYPES:
            raise SequenceError(f"unknown sequence dtype {dtype!r}")
        self.path = Path(path)
        self.path.mkdir(parents=True, exist_ok=True)
        self.width, self.height, self.dtype = int(width), int(height), dtype
        self.meta = dict(meta or {})
        self.count = 0
        self._frames: list[np.ndarray] = []
        self._fh = open(self.path / RAW_NAME, "wb") if dtype == "f32le" else None
        self.header: SequenceHeader | None = None

    def append(self, frame) -> None:
        frame = np.asarray(frame)
        if frame.shape != (self.height, self.width):
            raise SequenceError(f"frame shape {frame.shape} != {(self.height, self.width)}")
        if self._fh is not None:
            self._fh.write(np.ascontiguousarray(frame, dtype="<f4").data)
        else:
            self._frames.append(np.array(frame, dtype=np.float32))
        self.count += 1

    def close(self) -> SequenceHeader:
        if self.header is not None:
            return self.header
        if self._fh is not None:
            self._fh.close()
            hdr = SequenceHeader(self.width, self.height, self.count, "f32le", 1.0, 0.0, self.meta)
        else:
            stack = (np.stack(self._frames) if self._frames
                     else np.zeros((0, self.height, self.width), np.float32))
            scale, offset = _pgm_range(stack, None, None)
            hdr = SequenceHeader(self.width, self.height, self.count, "pgm16", scale, offset, self.meta)
            for i in range(self.count):
                with open(self.path / pgm_name(i), "wb") as fh:
                    fh.write(_pgm_bytes(stack[i], scale, offset))
            self._frames = []
        hdr.validate()
        _write_header(self.path, hdr)
        self.header = hdr
        return hdr

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
