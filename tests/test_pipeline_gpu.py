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


@pytest.mark.parametrize("world", [2, 4])
def test_strip_sharding_matches_full_frame(params, world):
    """The per-rank strip pipelines (halo rows + row offset, strips.py) stitch
    back to the full-frame result: emulated on one GPU by running every
    rank's local strip in turn (the halo rows are the ones exchange_halo
    delivers; the exchange itself is tested on gloo in test_strips_cpu)."""
    import torch

    from paper_1408_3526_b200 import Pipeline
    from paper_1408_3526_b200.strips import plan_strips

    rng = np.random.default_rng(world)
    t, h, w = 9, 96, 70
    frames = (10 + rng.standard_normal((t, h, w))).astype(np.float32)
    full, _, _ = _run_gpu(params, frames)
    plans = plan_strips(params, h, world)
    res = np.zeros((len(full), h, w), np.float32)
    idx = np.zeros((len(full), h, w, 2), np.int32)
    for pl in plans:
        with Pipeline(params, w, pl.local_height, _strip=(pl.halo, pl.lo)) as pipe:
            k = 0
            for n in range(t):
                o = pipe.process_frame_device(torch.from_numpy(frames[n, pl.lo:pl.a1]).cuda())
                if o is None:
                    continue
                mhy = params.mhat[1]
                r0 = pl.halo - mhy if pl.halo else 0
                res[k, pl.lo + r0: pl.a1 - mhy] = o.residual[r0: pl.local_height - mhy]
                idx[k, pl.a0:pl.a1] = o.velocity.indices[pl.halo:]
                k += 1
            assert k == len(full)
    fmax = float(np.abs(frames).max())
    for k, g in enumerate(full):
        assert velocity_agreement(idx[k], g.velocity.indices, params) >= VEL_FRAC
        m = g.mask & agreeing_outputs(idx[k], g.velocity.indices, params)
        assert residual_error(res[k], g.residual, m, fmax) <= RES_TOL


def test_device_frame_entry_matches_host_entry(params):
    import torch

    from paper_1408_3526_b200 import Pipeline

    rng = np.random.default_rng(3)
    frames = (10 + rng.standard_normal((8, 40, 50))).astype(np.float32)
    a, _, _ = _run_gpu(params, frames)
    with Pipeline(params, 50, 40) as pipe:
        b = [o for o in (pipe.process_frame_device(torch.from_numpy(f).cuda()) for f in frames) if o is not None]
    for x, y in zip(a, b):
        assert np.array_equal(x.residual, y.residual)
        assert np.array_equal(x.velocity.indices, y.velocity.indices)


def test_full_size_properties(params):
    """640x512 (config C3 geometry): DC-offset invariance of the residual and
    velocity agreement across offsets -- size-independent properties."""
    from paper_1408_3526_b200.scenegen import SimConfig, generate

    frames, _ = generate(SimConfig(width=640, height=512, frame_count=8, rng_seed=0))
    a, _, _ = _run_gpu(params, frames)
    b, _, _ = _run_gpu(params, frames + np.float32(5.0))
    for x, y in zip(a, b):
        m = x.mask & agreeing_outputs(x.velocity.indices, y.velocity.indices, params)
        assert np.abs(x.residual[m] - y.residual[m]).max() <= 1e-3 * 5.0
        assert velocity_agreement(x.velocity.indices, y.velocity.indices, params) >= 0.99


def test_full_size_crop_parity_vs_oracle(params):
    """640x512 C3 frames: the oracle on a 128x128 crop (plus the 8-px causal
    margin) against the same crop of the full-frame GPU run."""
    from paper_1408_3526_b200.scenegen import SimConfig, generate

    frames, _ = generate(SimConfig(width=640, height=512, frame_count=10, rng_seed=0))
    gpu, _, _ = _run_gpu(params, frames)
    y0, x0, n = 200, 300, 128
    crop = np.ascontiguousarray(frames[:, y0 - 8:y0 + n, x0 - 8:x0 + n])
    ref = _run_oracle(params, crop)
    fmax = float(np.abs(frames).max())
    for g, r in zip(gpu, ref):
        gi = g.velocity.indices[y0:y0 + n, x0:x0 + n]
        ri = r["indices"][8:, 8:]
        assert np.all(gi == ri, axis=-1).mean() >= VEL_FRAC
        # outputs of the crop's anchors sit at anchor - mhat = (-4, -4)
        same = np.all(gi == ri, axis=-1)
        gres = g.residual[y0 - 4:y0 + n - 4, x0 - 4:x0 + n - 4]
        rres = r["residual"][4:n + 4, 4:n + 4]
        assert np.abs(gres - rres)[same].max() / fmax <= RES_TOL


def test_process_stream_matches_process_frame(params):
    """The pipelined stream API (cw_submit/cw_wait, three streams) gives the
    same outputs as the synchronous call, frame for frame."""
    import torch

    from paper_1408_3526_b200 import Pipeline

    rng = np.random.default_rng(11)
    frames = (10 + rng.standard_normal((14, 48, 70))).astype(np.float32)
    pinned = torch.empty(frames.shape, dtype=torch.float32, pin_memory=True)
    pinned.copy_(torch.from_numpy(frames))
    a, _, _ = _run_gpu(params, frames)
    for depth in (1, 3, 6):
        with Pipeline(params, 70, 48) as pipe:
            b = list(pipe.process_stream(pinned.numpy(), depth=depth))
        assert [o.frame_index for o in b] == [o.frame_index for o in a]
        for x, y in zip(a, b):
            assert np.array_equal(x.residual, y.residual)
            assert np.array_equal(x.prediction, y.prediction)
            assert np.array_equal(x.velocity.indices, y.velocity.indices)
            assert np.array_equal(x.velocity.velocities, y.velocity.velocities)


def test_lazy_velocity_field_contract(params):
    """WhitenedOutput.velocity keeps the reference types (flow.py:134-144):
    int32 (H, W, 2) indices and float64 (H, W, 2) velocities = lag values."""
    rng = np.random.default_rng(12)
    frames = (10 + rng.standard_normal((7, 20, 24))).astype(np.float32)
    gpu, _, _ = _run_gpu(params, frames)
    v = gpu[-1].velocity
    assert v.indices.dtype == np.int32 and v.indices.shape == (20, 24, 2)
    assert v.velocities.dtype == np.float64 and v.velocities.shape == (20, 24, 2)
    lag = np.asarray(params.lag_grid_x)
    assert np.array_equal(v.velocities[..., 0], lag[v.indices[..., 0]])
    assert np.array_equal(v.velocities[..., 1], lag[v.indices[..., 1]])


@pytest.mark.parametrize("stream", [False, True])
def test_detection_epilogue_matches_host_metrics(params, stream):
    """Fused final threshold + metrics (cli.compute_metrics_row without
    truth, cli.py:157-208): peak |res| and its first row-major location over
    the valid mask, RMS over the mask, and every |res| >= tau."""
    from paper_1408_3526_b200 import Pipeline
    from paper_1408_3526_b200.scenegen import SimConfig, generate

    frames, _ = generate(SimConfig(width=96, height=80, frame_count=14, rng_seed=3))
    tau = 0.3
    with Pipeline(params, 96, 80, detect_threshold=tau, max_detections=4096) as pipe:
        outs = list(pipe.process_stream(frames)) if stream else \
            [o for o in (pipe.process_frame(f) for f in frames) if o is not None]
    assert len(outs) == 10
    for o in outs:
        m = o.metrics
        absres = np.abs(o.residual.astype(np.float64))
        masked = np.where(o.mask, absres, -1.0)
        py, px = np.unravel_index(int(np.argmax(masked)), absres.shape)
        assert (m["peak_x"], m["peak_y"]) == (px, py)
        assert m["peak_abs_residual"] == pytest.approx(absres[py, px], rel=1e-6)
        assert m["n_valid"] == int(o.mask.sum())
        rms = np.sqrt(np.mean(o.residual[o.mask].astype(np.float64) ** 2))
        assert m["residual_rms"] == pytest.approx(rms, rel=1e-5)
        ys, xs = np.nonzero(o.mask & (np.abs(o.residual) >= np.float32(tau)))
        assert m["n_detections"] == len(xs) and not m["truncated"]
        assert np.array_equal(o.detections[:, 0].astype(int), xs)
        assert np.array_equal(o.detections[:, 1].astype(int), ys)
        assert np.array_equal(o.detections[:, 2].astype(np.float32), o.residual[ys, xs])


def test_naive_backend_matches_recursive(params):
    """test_pipeline.py:131-139: the non-recursive spectrum backend gives the
    recursive pipeline's outputs (residual 1e-5, identical velocity bins)."""
    rng = np.random.default_rng(47)
    frames = rng.random((8, 14, 14)).astype(np.float32)
    rec, _, _ = _run_gpu(params, frames, spectrum_backend="recursive")
    nai, _, _ = _run_gpu(params, frames, spectrum_backend="naive")
    assert len(rec) == len(nai) == 4
    for a, b in zip(rec, nai):
        assert np.abs(a.residual - b.residual).max() < 1e-5
        assert np.array_equal(a.velocity.indices, b.velocity.indices)


def test_naive_backend_vs_oracle(params):
    from paper_1408_3526_b200.scenegen import SimConfig, generate

    frames, _ = generate(SimConfig(width=72, height=40, frame_count=12, rng_seed=8))
    gpu, specs, _ = _run_gpu(params, frames, spectrum_backend="naive", spectrum_at=(11,))
    _compare(params, frames, gpu, _run_oracle(params, frames))


@pytest.mark.parametrize("kw", [
    dict(lag_grid_x=(-1.0, -0.5, 0.25, 1.0, 1.75), lag_grid_y=(-1.25, 0.0, 0.5)),    # asymmetric grids
    dict(lag_grid_x=tuple(i / 4 - 0.125 for i in range(-7, 9)),                     # even length, no 0
         lag_grid_y=tuple(i / 4 - 0.125 for i in range(-7, 9))),
    dict(mhat=(0, 0, 0)),
    dict(mhat=(8, 8, 4)),
    dict(mhat=(2, 6, 1), alpha=0.5),
])
def test_parameter_variants_vs_oracle(kw):
    """The runtime-loop contraction (non-symmetric / even lag grids) and the
    output placement for other group delays, against the oracle."""
    from paper_1408_3526_b200 import FilterParams
    from paper_1408_3526_b200.scenegen import SimConfig, generate

    p = FilterParams(**kw)
    frames, _ = generate(SimConfig(width=70, height=45, frame_count=11, rng_seed=21))
    gpu, _, _ = _run_gpu(p, frames)
    _compare(p, frames, gpu, _run_oracle(p, frames))


def test_snapshot_restore_resumes_exactly(params):
    """Checkpoint after frame 7, restore into a fresh pipeline: frames 8.. give
    bit-identical outputs to the uninterrupted run (no new warm-up)."""
    from paper_1408_3526_b200 import Pipeline

    rng = np.random.default_rng(5)
    frames = (10 + rng.standard_normal((14, 40, 70))).astype(np.float32)
    full, _, _ = _run_gpu(params, frames)
    with Pipeline(params, 70, 40) as a:
        for f in frames[:8]:
            a.process_frame(f)
        snap = a.snapshot()
    with Pipeline(params, 70, 40) as b:
        b.restore(snap)
        assert b.frames_seen == 8
        resumed = [b.process_frame(f) for f in frames[8:]]
    for x, y in zip(full[-6:], resumed):
        assert y is not None and x.frame_index == y.frame_index
        assert np.array_equal(x.residual, y.residual)
        assert np.array_equal(x.velocity.indices, y.velocity.indices)
    with Pipeline(params, 71, 40) as c:
        with pytest.raises(ValueError):
            c.restore(snap)


def test_device_timing_reported(params):
    from paper_1408_3526_b200 import Pipeline

    rng = np.random.default_rng(6)
    with Pipeline(params, 64, 48, device_timing=True) as pipe:
        for f in (10 + rng.standard_normal((7, 48, 64))).astype(np.float32):
            pipe.process_frame(f)
        t = pipe.last_timings
    assert 0 < t["kernel"] <= t["pipeline"]


def test_host_buffer_kinds_give_identical_outputs(params):
    """cw_push's host paths: pageable or pinned input frame (staged copy vs
    direct DMA) and pageable or pinned output buffers (device-to-host copies
    vs the kernel writing into mapped host memory, border zeroed on the
    host) produce bit-identical outputs; dirty pinned buffers get their
    invalid border cleared."""
    import ctypes

    import torch

    from paper_1408_3526_b200 import Pipeline, _native
    from paper_1408_3526_b200.pipeline import valid_mask
    from paper_1408_3526_b200.scenegen import SimConfig, generate

    frames, _ = generate(SimConfig(width=72, height=40, frame_count=9, rng_seed=12))
    h, w = frames.shape[1:]
    lib = _native.load()
    mask = valid_mask(params, w, h)
    results = {}
    for in_pinned in (False, True):
        for out_pinned in (False, True):
            got = []
            with Pipeline(params, w, h) as pipe:
                for f in frames:
                    src = f
                    if in_pinned:
                        src = torch.from_numpy(f.copy()).pin_memory().numpy()
                    if out_pinned:
                        res = torch.full((h, w), 7.0, dtype=torch.float32).pin_memory().numpy()
                        pred = torch.full((h, w), 7.0, dtype=torch.float32).pin_memory().numpy()
                        vidx = torch.zeros((h, w, 2), dtype=torch.uint8).pin_memory().numpy()
                    else:
                        res = np.full((h, w), 7.0, np.float32)
                        pred = np.full((h, w), 7.0, np.float32)
                        vidx = np.zeros((h, w, 2), np.uint8)
                    ready, fidx = ctypes.c_int32(), ctypes.c_int64()
                    _native.check(lib.cw_push(pipe._h, _native.fptr(src), _native.fptr(res), _native.fptr(pred),
                                              vidx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                              ctypes.byref(ready), ctypes.byref(fidx), None), pipe._h)
                    if ready.value:
                        assert np.all(res[~mask] == 0) and np.all(pred[~mask] == 0)
                        got.append((int(fidx.value), res.copy(), pred.copy(), vidx.copy()))
            results[(in_pinned, out_pinned)] = got
    base = results[(False, False)]
    assert len(base) == frames.shape[0] - (params.mz - 1)
    for key, got in results.items():
        for a, b in zip(base, got):
            assert a[0] == b[0], key
            for x, y in zip(a[1:], b[1:]):
                assert np.array_equal(x, y), key


def test_push_rejects_device_buffers(params):
    """cw_push is the host-buffer call: device pointers fail with a status
    code and a message (cw_push_device is the device entry), no crash."""
    import ctypes

    import torch

    from paper_1408_3526_b200 import Pipeline, _native

    lib = _native.load()
    with Pipeline(params, 32, 24) as pipe:
        dev = torch.zeros((24, 32), dtype=torch.float32, device="cuda")
        r, f = ctypes.c_int32(), ctypes.c_int64()
        rc = lib.cw_push(pipe._h, dev.data_ptr(), None, None, None, ctypes.byref(r), ctypes.byref(f), None)
        assert rc == _native.CW_ERR_VALUE
        assert b"cw_push_device" in lib.cw_last_error(pipe._h)
        host = np.zeros((24, 32), np.float32)
        out = np.zeros((24, 32), np.float32)
        rc = lib.cw_push(pipe._h, host.ctypes.data, dev.data_ptr(), None, None, ctypes.byref(r), ctypes.byref(f), None)
        assert rc == _native.CW_ERR_VALUE
        assert pipe.process_frame(host) is None  # the pipeline still works
        del out


def test_long_chunks_recursive_vs_naive(params):
    """Tall frames give each CTA runs of ~280 rows, so the y-SDFT recursion
    runs 64 rows between direct restarts: against the non-recursive
    backend (every window summed directly, an on-device oracle for large
    frames) the velocity bins agree on >= 99.9% of anchors and the
    residuals to 1e-4 max|I| where they agree."""
    import torch

    from paper_1408_3526_b200 import Pipeline
    from paper_1408_3526_b200.scenegen import SimConfig, generate_device

    w, h = 1280, 2048
    frames = generate_device(SimConfig(width=w, height=h, frame_count=200, rng_seed=3), frames=8).cpu().numpy()
    outs = {}
    for backend in ("recursive", "naive"):
        with Pipeline(params, w, h, spectrum_backend=backend) as pipe:
            assert pipe.launch_info()["grid"] * 64 < (w // 32) * h  # chunks longer than a restart interval
            outs[backend] = [o for o in (pipe.process_frame(f) for f in frames) if o is not None]
        torch.cuda.empty_cache()
    fmax = float(np.abs(frames).max())
    for a, b in zip(outs["recursive"], outs["naive"]):
        assert velocity_agreement(a.velocity.indices, b.velocity.indices.astype(np.int32), params) >= VEL_FRAC
        m = a.mask & agreeing_outputs(a.velocity.indices, b.velocity.indices, params)
        assert residual_error(a.residual, b.residual, m, fmax) <= RES_TOL
