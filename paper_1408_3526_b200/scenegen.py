"""Synthetic cluttered IR sequences (the reference's input generator).

Restates /root/reference/pkg/src/clutterwhiten/scenegen.py: a rigid,
analytically translating sum of random low-frequency cosines over a DC
pedestal (generate, 152-209), an occluding Gaussian point target
(inject_target, 102-129) and white Gaussian noise drawn row-major in frame
order (add_noise, 132-139).  ``generate`` reproduces the reference bits
(same numpy RNG draw order; pinned by tests/test_host_layer.py against the
golden C1 frames).

``generate_device`` evaluates the same scene model on the GPU with a
hand-written kernel (csrc/cw_scene.cu) for benchmark-scale sequences: the
clutter components and target track are ``generate``'s, the noise is a
pure function of (seed, t, y, x) -- Philox4x32-10 + Box-Muller -- so any row
strip or crop of a frame equals the same pixels of the full frame for every
split (config C4 strips, crop oracles), and the optional non-uniform motion
field of SURVEY §8d config C2 is built in.  ``generate_counter`` is its
numpy twin: the same operation sequence in IEEE double (custom cos / exp /
log from +, -, *, / only), equal to the device output bit for bit.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["SimConfig", "generate", "generate_counter", "generate_device", "inject_target", "scene_components",
           "target_center"]


@dataclass(frozen=True)
class SimConfig:
    """Scene parameters; defaults are the reference simulation (scenegen.py:25-60)."""

    width: int = 64
    height: int = 64
    frame_count: int = 100
    clutter_velocity: tuple[float, float] = (1.625, 0.625)
    component_count: int = 25
    component_amplitude: float = 0.1
    freq_range: float = 2.0 / 9.0
    dc_offset: float = 10.0
    target_velocity: tuple[float, float] = (-0.625, -0.375)
    target_peak: float | None = 1.0
    psf_sigma: float = 1.0
    target_truncation: float = 0.1
    noise_sigma: float = 0.1
    rng_seed: int = 0

    def validate(self) -> None:
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be positive")
        if self.frame_count < 5:
            raise ValueError("frame_count must cover the temporal window (>= 5)")
        if self.component_count < 0:
            raise ValueError("component_count must be >= 0")
        if self.noise_sigma < 0:
            raise ValueError("noise_sigma must be >= 0")
        if self.target_peak is not None and self.target_peak <= self.target_truncation:
            raise ValueError("target peak must exceed the truncation threshold")
        if self.psf_sigma <= 0:
            raise ValueError("psf_sigma must be positive")


def target_center(cfg: SimConfig, t: int) -> tuple[float, float]:
    """Target centre at frame t; it reaches the image centre on the last frame."""
    last = cfg.frame_count - 1
    return (cfg.width / 2.0 + cfg.target_velocity[0] * (t - last),
            cfg.height / 2.0 + cfg.target_velocity[1] * (t - last))


def inject_target(frame, center, peak, sigma, truncation):
    """Replace pixels where the Gaussian blob clears ``truncation`` (in place)."""
    if peak <= truncation:
        raise ValueError("peak must exceed truncation")
    cx, cy = float(center[0]), float(center[1])
    h, w = frame.shape
    reach = sigma * math.sqrt(2.0 * math.log(peak / truncation))
    x0, x1 = max(0, int(math.floor(cx - reach))), min(w - 1, int(math.ceil(cx + reach)))
    y0, y1 = max(0, int(math.floor(cy - reach))), min(h - 1, int(math.ceil(cy + reach)))
    if x0 > x1 or y0 > y1:
        return frame
    gx = (np.arange(x0, x1 + 1, dtype=np.float64) - cx) ** 2
    gy = (np.arange(y0, y1 + 1, dtype=np.float64) - cy) ** 2
    blob = peak * np.exp(-(gx[None, :] + gy[:, None]) / (2.0 * sigma * sigma))
    win = frame[y0 : y1 + 1, x0 : x1 + 1]
    hit = blob >= truncation
    win[hit] = blob[hit].astype(win.dtype)
    return frame


def _components(cfg: SimConfig, rng) -> np.ndarray:
    comps = np.zeros((cfg.component_count, 4), dtype=np.float64)
    for i in range(cfg.component_count):
        comps[i, 0] = rng.uniform(-cfg.freq_range, cfg.freq_range)
        comps[i, 1] = rng.uniform(-cfg.freq_range, cfg.freq_range)
        comps[i, 2] = rng.uniform(0.0, 2.0 * math.pi)
        comps[i, 3] = cfg.component_amplitude
    return comps


def generate(cfg: SimConfig):
    """(frames (T, H, W) float32, components (N, 4)); reference-identical bits."""
    cfg.validate()
    rng = np.random.default_rng(cfg.rng_seed)
    comps = _components(cfg, rng)
    xs = np.arange(cfg.width, dtype=np.float64)[None, :]
    ys = np.arange(cfg.height, dtype=np.float64)[:, None]
    vx, vy = cfg.clutter_velocity
    frames = np.empty((cfg.frame_count, cfg.height, cfg.width), dtype=np.float32)
    acc = np.empty((cfg.height, cfg.width), dtype=np.float64)
    for t in range(cfg.frame_count):
        acc[:] = cfg.dc_offset
        for fx, fy, ph, amp in comps:
            acc += amp * np.cos(2.0 * math.pi * (fx * (xs - vx * t) + fy * (ys - vy * t)) + ph)
        if cfg.target_peak is not None:
            inject_target(acc, target_center(cfg, t), cfg.target_peak, cfg.psf_sigma, cfg.target_truncation)
        if cfg.noise_sigma > 0:
            acc += rng.normal(0.0, cfg.noise_sigma, size=acc.shape)
        frames[t] = acc.astype(np.float32)
    return frames, comps


# -- counter-based scene (csrc/cw_scene.cu and its numpy twin) ---------------

_TWO_PI = 6.283185307179586
_LN2_HI, _LN2_LO = 6.93147180369123816490e-01, 1.90821492927058770002e-10
_COS_C = [1.0 / 2432902008176640000.0, -1.0 / 6402373705728000.0, 1.0 / 20922789888000.0,
          -1.0 / 87178291200.0, 1.0 / 479001600.0, -1.0 / 3628800.0, 1.0 / 40320.0, -1.0 / 720.0,
          1.0 / 24.0, -0.5, 1.0]
_SIN_C = [-1.0 / 121645100408832000.0, 1.0 / 355687428096000.0, -1.0 / 1307674368000.0,
          1.0 / 6227020800.0, -1.0 / 39916800.0, 1.0 / 362880.0, -1.0 / 5040.0, 1.0 / 120.0,
          -1.0 / 6.0, 1.0]
_EXP_C = [1.0 / 355687428096000.0, 1.0 / 20922789888000.0, 1.0 / 1307674368000.0, 1.0 / 87178291200.0,
          1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0,
          1.0 / 40320.0, 1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0, 1.0]
_LOG_C = [1.0 / 23.0, 1.0 / 21.0, 1.0 / 19.0, 1.0 / 17.0, 1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0, 1.0 / 9.0,
          1.0 / 7.0, 1.0 / 5.0, 1.0 / 3.0, 1.0]


def _horner(coefs, x):
    p = np.full_like(x, coefs[0])
    for c in coefs[1:]:
        p = p * x + c
    return p


def _cos_turns(u):
    """cos(2 pi u), operation for operation as csrc/cw_scene.cu:cos_turns."""
    r = u - np.rint(u)
    q = np.rint(4.0 * r)
    s = r - 0.25 * q
    th = s * _TWO_PI
    t2 = th * th
    c = _horner(_COS_C, t2)
    sn = _horner(_SIN_C, t2) * th
    return np.where(q == 0.0, c, np.where(q == 1.0, -sn, np.where(q == -1.0, sn, -c)))


def _exp_nonpos(x):
    """exp(x), x <= 0, as csrc/cw_scene.cu:exp_nonpos."""
    k = np.rint(x * 1.4426950408889634)
    r = (x - k * _LN2_HI) - k * _LN2_LO
    p = _horner(_EXP_C, r)
    return np.where(x < -700.0, 0.0, np.ldexp(p, np.clip(k, -1100, 0).astype(np.int32)))


def _log_unit(u):
    """ln(u), 0 < u <= 1, as csrc/cw_scene.cu:log_unit."""
    m, e = np.frexp(u)
    low = m < 0.70710678118654752440
    m = np.where(low, m * 2.0, m)
    e = np.where(low, e - 1, e)
    s = (m - 1.0) / (m + 1.0)
    p = _horner(_LOG_C, s * s)
    de = e.astype(np.float64)
    return de * _LN2_HI + (2.0 * s * p + de * _LN2_LO)


def _philox4x32_10(c0, c1, c2, c3, key):
    """Philox4x32-10 on uint64 arrays holding 32-bit lanes."""
    m32 = np.uint64(0xFFFFFFFF)
    k0, k1 = key & 0xFFFFFFFF, (key >> 32) & 0xFFFFFFFF
    for _ in range(10):
        p0 = np.uint64(0xD2511F53) * c0
        p1 = np.uint64(0xCD9E8D57) * c2
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ np.uint64(k0)
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ np.uint64(k1)
        c0, c1, c2, c3 = n0, p1 & m32, n2, p0 & m32
        k0, k1 = (k0 + 0x9E3779B9) & 0xFFFFFFFF, (k1 + 0xBB67AE85) & 0xFFFFFFFF
    return c0, c1, c2, c3


def _scene_struct(cfg: SimConfig, nonuniform: bool, comps: np.ndarray):
    from . import _native

    sc = _native.cw_scene()
    sc.width, sc.height, sc.frame_count = cfg.width, cfg.height, cfg.frame_count
    sc.n_comp = comps.shape[0]
    sc.comps = comps.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double))
    sc.dc_offset = cfg.dc_offset
    sc.clutter_vx, sc.clutter_vy = cfg.clutter_velocity
    sc.nonuniform = int(bool(nonuniform))
    sc.motion_ax, sc.motion_ay = C2_MOTION
    sc.target = int(cfg.target_peak is not None)
    sc.target_vx, sc.target_vy = cfg.target_velocity
    sc.target_peak = cfg.target_peak if cfg.target_peak is not None else 0.0
    sc.psf_sigma, sc.target_truncation = cfg.psf_sigma, cfg.target_truncation
    sc.noise_sigma, sc.seed = cfg.noise_sigma, cfg.rng_seed
    return sc


#: config C2 motion-field amplitudes: v(x, y) = (vx + 0.5 sin(2 pi y / H), vy + 0.375 cos(2 pi x / W))
C2_MOTION = (0.5, 0.375)


def scene_components(cfg: SimConfig) -> np.ndarray:
    """(N, 4) fx, fy, phase, amplitude: the reference's first RNG draws
    (scenegen.py:169-175), shared by every generator here."""
    return np.ascontiguousarray(_components(cfg, np.random.default_rng(cfg.rng_seed)))


def generate_device(cfg: SimConfig, device="cuda", nonuniform: bool = False, frames: int | None = None,
                    rows: tuple[int, int] | None = None, cols: tuple[int, int] | None = None, t0: int = 0,
                    out=None):
    """Frames t0 .. t0+frames-1 of the counter-based scene on the GPU
    (csrc/cw_scene.cu), rows [r0, r1) and columns [c0, c1) of the full
    (H, W) frame, as a (T, r1-r0, c1-c0) float32 CUDA tensor (or into
    ``out``).  ``nonuniform`` adds the config-C2 motion field."""
    import torch

    from . import _native

    cfg.validate()
    comps = scene_components(cfg)
    n = cfg.frame_count - t0 if frames is None else int(frames)
    r0, r1 = rows if rows is not None else (0, cfg.height)
    c0, c1 = cols if cols is not None else (0, cfg.width)
    dev = torch.device(device)
    if out is None:
        out = torch.empty((n, r1 - r0, c1 - c0), dtype=torch.float32, device=dev)
    elif tuple(out.shape) != (n, r1 - r0, c1 - c0) or out.dtype != torch.float32 or not out.is_contiguous():
        raise ValueError("out must be a contiguous float32 tensor of the window shape")
    sc = _scene_struct(cfg, nonuniform, comps)
    lib = _native.load()
    with torch.cuda.device(out.device):
        stream = torch.cuda.current_stream(out.device).cuda_stream
        rc = lib.cw_scene_generate(__import__("ctypes").byref(sc), int(t0), n, r0, r1, c0, c1,
                                   out.data_ptr(), stream)
    if rc != 0:
        raise _native.NativeError(lib.cw_scene_last_error().decode())
    return out


def generate_counter(cfg: SimConfig, nonuniform: bool = False, frames: int | None = None,
                     rows: tuple[int, int] | None = None, cols: tuple[int, int] | None = None, t0: int = 0):
    """Host twin of ``generate_device``: the same (T, rows, cols) float32
    window, bit for bit (numpy, IEEE double, no FMA)."""
    cfg.validate()
    comps = scene_components(cfg)
    n = cfg.frame_count - t0 if frames is None else int(frames)
    r0, r1 = rows if rows is not None else (0, cfg.height)
    c0, c1 = cols if cols is not None else (0, cfg.width)
    xi = np.arange(c0, c1, dtype=np.int64)[None, :]
    yi = np.arange(r0, r1, dtype=np.int64)[:, None]
    xd, yd = xi.astype(np.float64), yi.astype(np.float64)
    shape = (r1 - r0, c1 - c0)
    vx = np.full(shape, float(cfg.clutter_velocity[0]))
    vy = np.full(shape, float(cfg.clutter_velocity[1]))
    if nonuniform:
        vx = vx + C2_MOTION[0] * _cos_turns(yd / float(cfg.height) - 0.25)
        vy = vy + C2_MOTION[1] * _cos_turns(xd / float(cfg.width))
    fx, fy = comps[:, 0], comps[:, 1]
    ph = comps[:, 2] / _TWO_PI
    amp = comps[:, 3]
    target = cfg.target_peak is not None
    if target:
        reach = cfg.psf_sigma * math.sqrt(2.0 * math.log(cfg.target_peak / cfg.target_truncation)) + 1.0
        two_s2 = 2.0 * cfg.psf_sigma * cfg.psf_sigma
    key = int(cfg.rng_seed) & 0xFFFFFFFFFFFFFFFF
    cx64 = np.broadcast_to(xi, shape).astype(np.uint64)
    cy64 = np.broadcast_to(yi, shape).astype(np.uint64)
    out = np.empty((n,) + shape, np.float32)
    for f in range(n):
        t = t0 + f
        td = float(t)
        px, py = xd - vx * td, yd - vy * td
        acc = np.full(shape, float(cfg.dc_offset))
        for i in range(comps.shape[0]):
            acc = acc + amp[i] * _cos_turns(fx[i] * px + fy[i] * py + ph[i])
        if target:
            tl = float(t - (cfg.frame_count - 1))
            tcx = cfg.width / 2.0 + cfg.target_velocity[0] * tl
            tcy = cfg.height / 2.0 + cfg.target_velocity[1] * tl
            dx, dy = xd - tcx, yd - tcy
            near = (np.abs(dx) <= reach) & (np.abs(dy) <= reach)
            if near.any():
                blob = cfg.target_peak * _exp_nonpos(-(dx * dx + dy * dy) / two_s2)
                acc = np.where(near & (blob >= cfg.target_truncation), blob, acc)
        if cfg.noise_sigma > 0:
            c2 = np.full(shape, t & 0xFFFFFFFF, np.uint64)
            c3 = np.full(shape, (t >> 32) & 0xFFFFFFFF, np.uint64)
            o0, o1, o2, o3 = _philox4x32_10(cx64, cy64, c2, c3, key)
            u1 = ((o0 >> np.uint64(5)).astype(np.float64) * 67108864.0
                  + (o1 >> np.uint64(6)).astype(np.float64) + 1.0) * 1.1102230246251565e-16
            u2 = ((o2 >> np.uint64(5)).astype(np.float64) * 67108864.0
                  + (o3 >> np.uint64(6)).astype(np.float64)) * 1.1102230246251565e-16
            z = np.sqrt(-2.0 * _log_unit(u1)) * _cos_turns(u2)
            acc = acc + cfg.noise_sigma * z
        out[f] = acc.astype(np.float32)
    return out
