"""Every validate-legal FilterParams runs on the device (params.py:114-158;
SPEC.md:69 makes the geometry runtime configuration).

Three device paths cover the domain: the fused instances compiled into the
library (kind 0); the same fused kernel compiled at run time by NVRTC for
any other geometry within its limits (kind 1: half windows <= 5, lag grids
<= 33 entries; cubins cached, csrc/cw_jit.cu); and the runtime-geometry
kernels (kind 2, csrc/cw_generic.cu) for everything else -- larger windows,
longer lag grids (more than 256 entries: uint16 indices).  Each is checked
against the float64 oracle / the reference's golden vectors with the
tolerances of tests/parity.py.  CW_NO_JIT=1 sends the kind-1 geometries to
the runtime-geometry kernels and CW_FORCE_GENERIC=1 the compiled ones, so
all paths are compared on the same parameter sets."""

import numpy as np
import pytest

from conftest import SMALL_CASES, small_case
from parity import RES_TOL, VEL_FRAC, agreeing_outputs, residual_error, velocity_agreement

pytestmark = pytest.mark.gpu


def _frames(t, h, w, seed=0, vx=1.25, vy=0.5):
    rng = np.random.default_rng(seed)
    xs, ys = np.arange(w)[None, :], np.arange(h)[:, None]
    return np.stack([
        10.0 + 0.3 * np.cos(2 * np.pi * ((xs - vx * n) / 9.0 + (ys - vy * n) / 7.0))
        + 0.2 * np.cos(2 * np.pi * ((xs - vx * n) / 13.0 - (ys - vy * n) / 11.0))
        + 0.05 * rng.standard_normal((h, w)) for n in range(t)
    ]).astype(np.float32)


def _check(params, frames, gpu_outs, ref_outs):
    assert len(gpu_outs) == len(ref_outs) > 0
    fmax = float(np.abs(frames).max())
    for g, r in zip(gpu_outs, ref_outs):
        assert g.frame_index == r["frame_index"]
        assert velocity_agreement(g.velocity.indices, r["indices"], params) >= VEL_FRAC
        m = g.mask & agreeing_outputs(g.velocity.indices, r["indices"], params)
        if m.any():
            assert residual_error(g.residual, r["residual"], m, fmax) <= RES_TOL
        assert np.all(g.residual[~g.mask] == 0)


def _run(params, frames, **kw):
    """(outputs, ran the runtime-geometry kernels)"""
    outs, kind = _run_kind(params, frames, **kw)
    return outs, kind == 2


def _run_kind(params, frames, **kw):
    from paper_1408_3526_b200 import Pipeline, _native

    t, h, w = frames.shape
    with Pipeline(params, w, h, **kw) as pipe:
        outs = [o for o in map(pipe.process_frame, frames) if o is not None]
        kind = int(_native.load().cw_kernel_kind(pipe._h))
        assert bool(_native.load().cw_is_generic(pipe._h)) == (kind == 2)
        assert pipe.kernel_kind == ("compiled", "jit", "runtime-geometry")[kind]
    return outs, kind


def _oracle(params, frames, forced=None):
    from oracle.oracle import OraclePipeline

    t, h, w = frames.shape
    with OraclePipeline(params, w, h, forced_velocity=forced) as orc:
        return [o for o in map(orc.process_frame, frames) if o is not None]


@pytest.mark.parametrize("name", SMALL_CASES)
def test_generic_path_on_the_golden_cases(name, monkeypatch):
    """The reference's own outputs (tests/golden/small_cases.npz) through the
    runtime-geometry kernels."""
    monkeypatch.setenv("CW_FORCE_GENERIC", "1")
    p, frames, forced, want = small_case(name)
    outs, generic = _run(p, frames, forced_velocity=forced)
    assert generic
    ref = [{"frame_index": int(want["frame_index"][k]), "indices": want["indices"][k],
            "residual": want["residual"][k]} for k in range(len(want["frame_index"]))]
    _check(p, frames, outs, ref)


LEGAL = {
    # (kx, ky, kz, bx, by, mhat, lag_x, lag_y): none has an instance compiled
    # into the library
    "bx2": (4, 4, 2, 2, 3, (4, 4, 2), None, None),
    "kz3": (4, 4, 3, 3, 3, (4, 4, 3), None, None),
    "ky3_by2": (4, 3, 2, 3, 2, (4, 3, 2), None, None),
    "k6": (6, 6, 2, 5, 5, (6, 6, 2), None, None),
    "k1_b0": (1, 1, 1, 0, 0, (1, 1, 1), (-0.5, 0.0, 0.5), (-1.0, 0.0, 1.0)),
    "k2_mhat0": (2, 3, 1, 1, 2, (0, 1, 0), None, None),
    "lags41_asym": (4, 4, 2, 3, 3, (4, 4, 2), tuple(-2.0 + 0.1 * i for i in range(41)),
                    tuple(-1.5 + 0.125 * i for i in range(25))),
    "lags_even": (4, 4, 2, 3, 3, (4, 4, 2), (-1.5, -0.5, 0.5, 1.5), (-1.0, 0.0, 0.75)),
}


def _params(spec):
    from paper_1408_3526_b200 import FilterParams, validate

    kx, ky, kz, bx, by, mhat, lx, ly = spec
    kw = dict(kx=kx, ky=ky, kz=kz, bx=bx, by=by, mhat=mhat)
    if lx is not None:
        kw.update(lag_grid_x=lx, lag_grid_y=ly)
    elif min(kx, ky) < 2:
        kw.update(lag_grid_x=(-1.0, 0.0, 1.0), lag_grid_y=(-1.0, 0.0, 1.0))
    p = FilterParams(**kw)
    validate(p)
    return p


# kind each set runs with NVRTC available: beyond the fused kernel's limits
# (K = 6, 41 lags) -> runtime-geometry kernels; a short lag grid on the
# compiled default geometry -> the compiled runtime-loop instance
EXPECTED_KIND = {"k6": 2, "lags41_asym": 2, "lags_even": 0}


@pytest.mark.parametrize("path", ["fused", "runtime_geometry"])
@pytest.mark.parametrize("name", sorted(LEGAL))
def test_legal_geometry_matches_oracle(name, path, monkeypatch):
    if path == "runtime_geometry":
        monkeypatch.setenv("CW_NO_JIT", "1")
    p = _params(LEGAL[name])
    h, w = 2 * p.my + 22, 2 * p.mx + 31
    frames = _frames(p.mz + 7, h, w, seed=len(name))
    outs, kind = _run_kind(p, frames)
    want = EXPECTED_KIND.get(name, 1)
    assert kind == (2 if path == "runtime_geometry" and want == 1 else want)
    _check(p, frames, outs, _oracle(p, frames))


def test_jit_instance_equals_generic_on_the_same_geometry(monkeypatch):
    """The run-time compiled fused kernel and the runtime-geometry kernels on
    one non-compiled geometry: the same velocities up to near-ties."""
    p = _params(LEGAL["kz3"])
    frames = _frames(14, 60, 72, seed=12)
    fused, k1 = _run_kind(p, frames)
    monkeypatch.setenv("CW_NO_JIT", "1")
    gen, k2 = _run_kind(p, frames)
    assert (k1, k2) == (1, 2)
    fmax = float(np.abs(frames).max())
    for a, b in zip(fused, gen):
        assert velocity_agreement(a.velocity.indices, b.velocity.indices, p) >= VEL_FRAC
        m = a.mask & agreeing_outputs(a.velocity.indices, b.velocity.indices, p)
        assert residual_error(a.residual, b.residual.astype(np.float64), m, fmax) <= RES_TOL


def test_more_than_256_lags_use_16_bit_indices():
    """A 260-entry lag grid (legal: params.py:142-157 bounds only the span)
    returns indices > 255: the device writes uint16 pairs."""
    from paper_1408_3526_b200 import FilterParams

    from oracle.oracle import OraclePipeline

    lx = tuple(float(v) for v in np.linspace(-3.9, 3.9, 260))
    p = FilterParams(lag_grid_x=lx, lag_grid_y=(-0.5, 0.0, 0.5))
    frames = _frames(9, 40, 48, seed=9, vx=1.3, vy=0.1)
    outs, generic = _run(p, frames)
    assert generic
    gx = 0.375 / (0.25 + 0.125 * np.cos(2 * np.pi * np.asarray(lx) / p.mx))
    gy = 0.375 / (0.25 + 0.125 * np.cos(2 * np.pi * np.asarray(p.lag_grid_y) / p.my))
    fmax = float(np.abs(frames).max())
    with OraclePipeline(p, 48, 40) as orc:
        k = 0
        for f in frames:
            r = orc.process_frame(f)
            if r is None:
                continue
            g = outs[k]
            k += 1
            # lag steps of 0.03 px put neighbouring scores within f32 rounding:
            # every disagreement must be a near-tie of the oracle's own scores
            score = orc.rhat() * gy[None, None, :, None] * gx[None, None, None, :]
            gi, ri = g.velocity.indices, r["indices"]
            ys, xs = np.nonzero(np.any(gi != ri, axis=-1))
            for y, x in zip(ys, xs):
                mine, theirs = score[y, x, gi[y, x, 1], gi[y, x, 0]], score[y, x, ri[y, x, 1], ri[y, x, 0]]
                assert theirs - mine <= 2e-5 * abs(theirs), (y, x)
            assert velocity_agreement(gi, ri, p) >= 0.995
            m = g.mask & agreeing_outputs(gi, ri, p)
            assert residual_error(g.residual, r["residual"], m, fmax) <= RES_TOL
        assert k == len(outs)
    v = outs[-1].velocity
    assert np.array_equal(v.velocities[..., 0], np.asarray(lx)[v.indices[..., 0]])
    # indices past 255 survive the device -> host path (uint16 pairs)
    forced, _ = _run(p, frames, forced_velocity=(lx[258], 0.5))
    assert np.all(forced[-1].velocity.indices == (258, 2))
    assert np.all(forced[-1].velocity.velocities == (lx[258], 0.5))
    ref = _oracle(p, frames, forced=(lx[258], 0.5))
    assert np.abs(forced[-1].residual - ref[-1]["residual"]).max() <= RES_TOL * fmax


def test_generic_equals_fused_on_the_default_geometry(params, monkeypatch):
    """Same frames through the fused kernel and (forced) the runtime path."""
    frames = _frames(12, 70, 90, seed=3)
    fused, g0 = _run(params, frames)
    monkeypatch.setenv("CW_FORCE_GENERIC", "1")
    gen, g1 = _run(params, frames)
    assert not g0 and g1
    fmax = float(np.abs(frames).max())
    for a, b in zip(fused, gen):
        assert velocity_agreement(a.velocity.indices, b.velocity.indices, params) >= VEL_FRAC
        m = a.mask & agreeing_outputs(a.velocity.indices, b.velocity.indices, params)
        assert residual_error(a.residual, b.residual.astype(np.float64), m, fmax) <= RES_TOL


@pytest.mark.parametrize("path", ["fused", "runtime_geometry"])
def test_generic_naive_backend_forced_velocity_and_detection(path, monkeypatch):
    """The naive spectrum backend, forced velocity and the detection metrics
    (pipeline.py:139-142, 174-177, 260-265) on a non-compiled geometry, run
    time compiled and on the runtime-geometry kernels."""
    if path == "runtime_geometry":
        monkeypatch.setenv("CW_NO_JIT", "1")
    p = _params(LEGAL["kz3"])
    frames = _frames(11, 40, 44, seed=4)
    ref = _oracle(p, frames)
    outs, kind = _run_kind(p, frames, spectrum_backend="naive", detect_threshold=0.05)
    assert kind == (1 if path == "fused" else 2)
    _check(p, frames, outs, ref)
    for o in outs:
        want = np.sqrt(np.mean(o.residual[o.mask].astype(np.float64) ** 2))
        assert o.metrics["residual_rms"] == pytest.approx(want, rel=1e-12)
        assert o.metrics["n_valid"] == int(o.mask.sum())
    forced = (p.lag_grid_x[2], p.lag_grid_y[5])
    outs, _ = _run(p, frames, forced_velocity=forced)
    _check(p, frames, outs, _oracle(p, frames, forced=forced))
    assert np.all(outs[-1].velocity.indices == (2, 5))


@pytest.mark.parametrize("path", ["fused", "runtime_geometry"])
def test_generic_strips_stitch_to_the_full_frame(path, monkeypatch):
    """Strip sharding (halo rows + row offset, strips.py) on a non-compiled
    geometry, both paths."""
    if path == "runtime_geometry":
        monkeypatch.setenv("CW_NO_JIT", "1")
    import torch

    from paper_1408_3526_b200 import Pipeline
    from paper_1408_3526_b200.strips import plan_strips

    p = _params(LEGAL["ky3_by2"])
    frames = _frames(9, 60, 50, seed=6)
    full, _ = _run(p, frames)
    for pl in plan_strips(p, 60, 3):
        with Pipeline(p, 50, pl.local_height, _strip=(pl.halo, pl.lo)) as pipe:
            k = 0
            for f in frames:
                o = pipe.process_frame_device(torch.from_numpy(f[pl.lo:pl.a1]).cuda())
                if o is None:
                    continue
                g = full[k]
                k += 1
                assert np.array_equal(o.velocity.indices[pl.halo:], g.velocity.indices[pl.a0:pl.a1])
                mhy = p.mhat[1]
                r0 = pl.halo - mhy if pl.halo else 0
                np.testing.assert_array_equal(o.residual[r0:pl.local_height - mhy],
                                              g.residual[pl.lo + r0:pl.a1 - mhy])


@pytest.mark.parametrize("path", ["fused", "runtime_geometry"])
def test_generic_snapshot_and_views(path, monkeypatch):
    """Checkpoint / resume and the spectrum / T^ parity views on a
    non-compiled geometry, both paths (the spectrum against the oracle's,
    per pixel)."""
    if path == "runtime_geometry":
        monkeypatch.setenv("CW_NO_JIT", "1")
    from oracle.oracle import OraclePipeline
    from paper_1408_3526_b200 import Pipeline
    from parity import SPEC_TOL, per_pixel_rel

    p = _params(LEGAL["bx2"])
    frames = _frames(10, 30, 34, seed=8)
    with Pipeline(p, 34, 30) as a, OraclePipeline(p, 34, 30) as orc:
        for f in frames[:7]:
            a.process_frame(f)
            orc.process_frame(f)
        err = per_pixel_rel(a.spectrum()[p.my - 1:, p.mx - 1:], orc.sbins()[p.my - 1:, p.mx - 1:], axes=(2, 3, 4))
        assert err <= SPEC_TOL
        assert a.smoothed_state().shape == (30, 34, p.my, p.mx)
        snap = a.snapshot()
        rest_a = [a.process_frame(f) for f in frames[7:]]
    with Pipeline(p, 34, 30) as b:
        b.restore(snap)
        rest_b = [b.process_frame(f) for f in frames[7:]]
    for x, y in zip(rest_a, rest_b):
        assert np.array_equal(x.residual, y.residual)
        assert np.array_equal(x.velocity.indices, y.velocity.indices)
