"""Synthetic cluttered IR sequences (the reference's input generator).

Restates /root/reference/pkg/src/clutterwhiten/scenegen.py: a rigid,
analytically translating sum of random low-frequency cosines over a DC
pedestal (generate, 152-209), an occluding Gaussian point target
(inject_target, 102-129) and white Gaussian noise drawn row-major in frame
order (add_noise, 132-139).  ``generate`` reproduces the reference bits
(same numpy RNG draw order; pinned by tests/test_host_layer.py against the
golden C1 frames).

``generate_device`` evaluates the same analytic model on the GPU (float64
cosines, torch) for benchmark-scale sequences; its clutter components and
target track are identical to ``generate``'s, its noise comes from torch's
counter-based CUDA generator (same distribution, different bits), and it
optionally adds the non-uniform motion field of SURVEY §8d config C2.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["SimConfig", "generate", "generate_device", "inject_target", "target_center"]


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


def generate_device(cfg: SimConfig, device="cuda", nonuniform: bool = False, frames: int | None = None,
                    rows: tuple[int, int] | None = None):
    """Same scene model evaluated on the GPU (torch float64), returns a
    (T, H, W) float32 CUDA tensor.  ``nonuniform`` applies the config-C2
    motion field v(x, y) = (vx + 0.5 sin(2 pi y / H), vy + 0.375 cos(2 pi x / W)).
    ``rows=(r0, r1)`` evaluates only image rows [r0, r1) (a strip of a large
    frame, e.g. one rank's share of config C4); noise is drawn per strip."""
    import torch

    cfg.validate()
    rng = np.random.default_rng(cfg.rng_seed)
    comps = torch.tensor(_components(cfg, rng), dtype=torch.float64, device=device)
    n_frames = cfg.frame_count if frames is None else int(frames)
    r0, r1 = rows if rows is not None else (0, cfg.height)
    h, w = r1 - r0, cfg.width
    xs = torch.arange(w, dtype=torch.float64, device=device)[None, :]
    ys = torch.arange(r0, r1, dtype=torch.float64, device=device)[:, None]
    vx = torch.full((h, w), cfg.clutter_velocity[0], dtype=torch.float64, device=device)
    vy = torch.full((h, w), cfg.clutter_velocity[1], dtype=torch.float64, device=device)
    if nonuniform:
        vx = vx + 0.5 * torch.sin(2 * math.pi * ys / cfg.height)
        vy = vy + 0.375 * torch.cos(2 * math.pi * xs / cfg.width)
    gen = torch.Generator(device=device)
    gen.manual_seed(cfg.rng_seed * 1000003 + r0)
    out = torch.empty((n_frames, h, w), dtype=torch.float32, device=device)
    for t in range(n_frames):
        acc = torch.full((h, w), cfg.dc_offset, dtype=torch.float64, device=device)
        px, py = xs - vx * t, ys - vy * t
        for fx, fy, ph, amp in comps:
            acc += amp * torch.cos(2.0 * math.pi * (fx * px + fy * py) + ph)
        if cfg.target_peak is not None:
            cx, cy = target_center(cfg, t)
            r2 = (xs - cx) ** 2 + (ys - cy) ** 2
            blob = cfg.target_peak * torch.exp(-r2 / (2.0 * cfg.psf_sigma ** 2))
            acc = torch.where(blob >= cfg.target_truncation, blob, acc)
        if cfg.noise_sigma > 0:
            acc += cfg.noise_sigma * torch.randn((h, w), dtype=torch.float64, device=device, generator=gen)
        out[t] = acc.to(torch.float32)
    return out
