"""Counter-based scene generator (csrc/cw_scene.cu + scenegen.generate_counter).

CPU: the numpy twin against a plain restatement of the scene model (numpy
cos / exp, the reference's formula, scenegen.py:152-209, plus the config-C2
motion field of SURVEY §8d), window invariance and noise statistics.
GPU: the device kernel equals the twin bit for bit, and any strip split or
crop of a frame equals the same pixels of the full frame."""

import math

import numpy as np
import pytest


def _model(cfg, t, nonuniform, noise=False):
    """The scene model in plain numpy (float64 cos / exp), no noise."""
    from paper_1408_3526_b200.scenegen import C2_MOTION, scene_components, target_center

    comps = scene_components(cfg)
    xs = np.arange(cfg.width, dtype=np.float64)[None, :]
    ys = np.arange(cfg.height, dtype=np.float64)[:, None]
    vx = np.full((cfg.height, cfg.width), cfg.clutter_velocity[0])
    vy = np.full((cfg.height, cfg.width), cfg.clutter_velocity[1])
    if nonuniform:
        vx = vx + C2_MOTION[0] * np.sin(2 * np.pi * ys / cfg.height)
        vy = vy + C2_MOTION[1] * np.cos(2 * np.pi * xs / cfg.width)
    acc = np.full((cfg.height, cfg.width), cfg.dc_offset)
    for fx, fy, ph, amp in comps:
        acc += amp * np.cos(2 * np.pi * (fx * (xs - vx * t) + fy * (ys - vy * t)) + ph)
    if cfg.target_peak is not None:
        cx, cy = target_center(cfg, t)
        blob = cfg.target_peak * np.exp(-((xs - cx) ** 2 + (ys - cy) ** 2) / (2 * cfg.psf_sigma ** 2))
        acc = np.where(blob >= cfg.target_truncation, blob, acc)
    return acc


@pytest.mark.parametrize("nonuniform", [False, True])
def test_twin_is_the_scene_model(nonuniform):
    from paper_1408_3526_b200.scenegen import SimConfig, generate_counter

    cfg = SimConfig(width=96, height=80, frame_count=12, rng_seed=2, noise_sigma=0.0)
    got = generate_counter(cfg, nonuniform=nonuniform, frames=4, t0=8)
    for k in range(4):
        want = _model(cfg, 8 + k, nonuniform)
        assert np.abs(got[k] - want).max() <= 2e-6 * np.abs(want).max()
    # the target is in the last frame at the image centre (scenegen.py:141-149)
    assert got[-1][40, 48] == pytest.approx(cfg.target_peak, abs=1e-6)


def test_twin_windows_are_the_full_frame_pixels():
    from paper_1408_3526_b200.scenegen import SimConfig, generate_counter

    cfg = SimConfig(width=70, height=64, frame_count=9, rng_seed=5)
    full = generate_counter(cfg, nonuniform=True, frames=3, t0=2)
    for rows, cols in (((0, 64), (0, 70)), ((13, 40), (0, 70)), ((5, 6), (33, 69)), ((60, 64), (1, 2))):
        part = generate_counter(cfg, nonuniform=True, frames=2, rows=rows, cols=cols, t0=3)
        assert np.array_equal(part, full[1:3, rows[0]:rows[1], cols[0]:cols[1]])


def test_twin_noise_is_white_gaussian():
    from paper_1408_3526_b200.scenegen import SimConfig, generate_counter

    cfg = SimConfig(width=256, height=128, frame_count=6, rng_seed=11, component_count=0, target_peak=None,
                    noise_sigma=1.0, dc_offset=0.0)
    z = generate_counter(cfg, frames=4).astype(np.float64)
    n = z.size
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.std() - 1.0) < 0.01
    assert abs((z ** 4).mean() - 3.0) < 0.05
    # no correlation between neighbours in x, y or t
    for a, b in ((z[:, :, 1:], z[:, :, :-1]), (z[:, 1:], z[:, :-1]), (z[1:], z[:-1])):
        assert abs(np.corrcoef(a.ravel(), b.ravel())[0, 1]) < 0.01
    # another seed gives another realisation
    other = generate_counter(SimConfig(**{**cfg.__dict__, "rng_seed": 12}), frames=1)
    assert not np.array_equal(other[0], z[0].astype(np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("nonuniform", [False, True])
def test_device_equals_twin_bit_for_bit(nonuniform):
    from paper_1408_3526_b200.scenegen import SimConfig, generate_counter, generate_device

    cfg = SimConfig(width=160, height=96, frame_count=40, rng_seed=7)
    dev = generate_device(cfg, nonuniform=nonuniform, frames=5, t0=30).cpu().numpy()
    host = generate_counter(cfg, nonuniform=nonuniform, frames=5, t0=30)
    assert np.array_equal(dev, host)
    crop = generate_device(cfg, nonuniform=nonuniform, frames=2, rows=(17, 60), cols=(9, 141), t0=32).cpu().numpy()
    assert np.array_equal(crop, host[2:4, 17:60, 9:141])


@pytest.mark.gpu
def test_device_strips_are_split_invariant():
    """Config C4: a rank's strip equals the same rows of the full frame for
    N = 1 / 2 / 4 / 8 strips (plus the 8-row halo above each strip)."""
    import torch

    from paper_1408_3526_b200.scenegen import SimConfig, generate_device

    cfg = SimConfig(width=512, height=512, frame_count=200, rng_seed=4)
    full = generate_device(cfg, frames=3, t0=100)
    for n in (2, 4, 8):
        rows = 512 // n
        for g in range(n):
            r0, r1 = max(0, g * rows - 8), (g + 1) * rows
            part = generate_device(cfg, frames=3, t0=100, rows=(r0, r1))
            assert torch.equal(part, full[:, r0:r1])
