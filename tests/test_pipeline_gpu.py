"""GPU parity: the fused sm_100a path (through the C ABI) against the
float64 oracle, which tests/test_oracle_golden.py pins bit-exactly to the
reference.  Tolerances are those of tests/parity.py."""

import numpy as np
import pytest

from conftest import SMALL_CASES, golden, small_case
from parity import (
    RES_TOL, RHAT_TOL, SPEC_TOL, VEL_FRAC, agreeing_outputs, per_pixel_rel, residual_error,
    velocity_agreement,
)

pytestmark = pytest.mark.gpu


def _run_gpu(params, frames, forced=None, bank=None, spectrum_at=(), **kw):
    from paper_1408_3526_b200 import Pipeline

    t, h, w = frames.shape
    outs, specs, thats = [], {}, {}
    with Pipeline(params, w, h, forced_velocity=forced, bank=bank, **kw) as pipe:
        if spectrum_at:
            pipe.enable_spectrum_dump()
        for n in range(t):
            o = pipe.process_frame(frames[n])
            if o is not None:
                outs.append(o)
            if n in spectrum_at:
                specs[n] = pipe.spectrum()
                thats[n] = pipe.smoothed_state()
    return outs, specs, thats


def _run_oracle(params, frames, forced=None):
    from oracle.oracle import OraclePipeline

    t, h, w = frames.shape
    with OraclePipeline(params, w, h, forced_velocity=forced) as orc:
        return [o for o in (orc.process_frame(f) for f in frames) if o is not None]


def _compare(params, frames, gpu, ref, vel_frac=VEL_FRAC):
    assert len(gpu) == len(ref)
    fmax = float(np.abs(frames).max())
    for g, r in zip(gpu, ref):
        assert g.frame_index == r["frame_index"]
        assert velocity_agreement(g.velocity.indices, r["indices"], params) >= vel_frac
        # residual parity where the velocity agrees (a flipped near-tie picks
        # a different, equally valid predictor)
        m = g.mask & agreeing_outputs(g.velocity.indices, r["indices"], params)
        if m.any():
            assert residual_error(g.residual, r["residual"], m, fmax) <= RES_TOL
        assert np.all(g.residual[~g.mask] == 0)
        assert np.all(g.prediction[~g.mask] == 0)
        assert g.imag_peak < 1e-6


def test_c1_golden_parity(params):
    """Config C1 (64x64x32, reference generator): every output frame."""
    z = golden("c1_64x64x32.npz")
    frames = z["frames"]
    gpu, specs, thats = _run_gpu(params, frames, spectrum_at=tuple(int(v) for v in z["crop_frames"]))
    assert len(gpu) == 28
    ref = [
        {"frame_index": int(z["frame_index"][k]), "residual": z["residual"][k],
         "indices": z["indices"][k].astype(np.int32)}
        for k in range(28)
    ]
    _compare(params, frames, gpu, ref)
    from paper_1408_3526_b200.pipeline import rhat_from_state

    y0, y1, x0, x1 = (int(v) for v in z["crop_box"])
    for j, n in enumerate(int(v) for v in z["crop_frames"]):
        s = specs[n][y0:y1, x0:x1]
        assert per_pixel_rel(s, z["spec_crops"][j], axes=(-3, -2, -1)) <= SPEC_TOL
        rh = rhat_from_state(thats[n][y0:y1, x0:x1], params)
        assert per_pixel_rel(rh, z["rhat_crops"][j], axes=(-2, -1)) <= RHAT_TOL


@pytest.mark.parametrize("name", SMALL_CASES)
def test_small_golden_cases(name):
    p, frames, forced, outs = small_case(name)
    gpu, _, _ = _run_gpu(p, frames, forced=forced)
    ref = [
        {"frame_index": int(outs["frame_index"][k]), "residual": outs["residual"][k],
         "indices": outs["indices"][k].astype(np.int32)}
        for k in range(len(outs["residual"]))
    ]
    _compare(p, frames, gpu, ref)


@pytest.mark.parametrize("shape", [(14, 9, 9), (12, 40, 33), (10, 70, 97), (9, 130, 200)])
def test_random_frames_vs_oracle(params, shape):
    """Ragged widths (partial 32-column blocks), minimum-size images and
    heights that cross the y-SDFT restart interval and CTA chunk edges."""
    rng = np.random.default_rng(sum(shape))
    frames = (10 + rng.standard_normal(shape)).astype(np.float32)
    gpu, _, _ = _run_gpu(params, frames)
    _compare(params, frames, gpu, _run_oracle(params, frames))


def test_scene_sequence_vs_oracle(params):
    """Longer reference-generator sequence: observer + smoothing over 40 frames."""
    z = golden("c1_64x64x32.npz")
    rng = np.random.default_rng(9)
    frames = np.concatenate([z["frames"], z["frames"][::-1]])[:40]
    frames = frames + rng.normal(0, 0.01, frames.shape).astype(np.float32)
    gpu, _, _ = _run_gpu(params, frames)
    _compare(params, frames, gpu, _run_oracle(params, frames))


def test_forced_velocity_reported(params):
    rng = np.random.default_rng(49)
    frames = rng.random((6, 16, 16)).astype(np.float32)
    gpu, _, _ = _run_gpu(params, frames, forced=(1.0, -0.5))
    assert np.all(gpu[0].velocity.velocities[..., 0] == 1.0)
    assert np.all(gpu[0].velocity.velocities[..., 1] == -0.5)


def test_constant_input_residual_vanishes(params):
    frames = np.full((10, 40, 70), 10.0, dtype=np.float32)
    gpu, _, _ = _run_gpu(params, frames)
    for o in gpu:
        assert np.abs(o.residual[o.mask]).max() < 1e-3
        assert np.abs(o.prediction[o.mask] - 10.0).max() < 1e-3
        # all-zero flow surface: ties resolve to the zero-velocity bin
        assert np.all(o.velocity.indices[8:, 8:] == 8)


def test_model_null_forced_velocity(params):
    """Acceptance 5 (test_acceptance.py:130-158): in-band translating cosine."""
    vx, vy = 1.0, 0.5
    xs, ys = np.arange(64)[None, :], np.arange(64)[:, None]
    frames = np.stack([np.cos(2 * np.pi * ((xs - vx * t) / 9 + 2 * (ys - vy * t) / 9)) for t in range(12)])
    gpu, _, _ = _run_gpu(params, frames.astype(np.float32), forced=(vx, vy))
    res = np.concatenate([o.residual[o.mask] for o in gpu]).astype(np.float64)
    assert np.sqrt(np.mean(res ** 2)) < 0.01


def test_outputs_are_fresh_copies(params):
    from paper_1408_3526_b200 import Pipeline

    rng = np.random.default_rng(46)
    frames = rng.random((7, 16, 16)).astype(np.float32)
    keep = []
    with Pipeline(params, 16, 16) as pipe:
        for f in frames:
            o = pipe.process_frame(f)
            if o is not None:
                keep.append((o, o.residual.copy()))
    for o, snap in keep:
        assert np.array_equal(o.residual, snap)
