"""Frame chaining: consecutive frame kernels overlap
(programmatic dependent launch, per-CTA completion flags, flagged
copy-engine ring copies for resident frames, stream-memory-write flags for
cw_submit uploads and downloads).  The
chained entry points must give bit-identical results to plain, fully
serialised launches with the same (static) work split, across frame sizes
whose CTA runs are short (C2-like) and long, mixed entry points, and a
snapshot restore in the middle of a chained stream."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _frames(t, h, w, seed=0):
    rng = np.random.default_rng(seed)
    xs, ys = np.arange(w)[None, :], np.arange(h)[:, None]
    return np.stack([
        10.0 + 0.3 * np.cos(2 * np.pi * ((xs - 1.25 * n) / 9.0 + (ys - 0.5 * n) / 7.0))
        + 0.05 * rng.standard_normal((h, w)) for n in range(t)
    ]).astype(np.float32)


def _dev_outputs(lib, pipe, native):
    w, h = pipe.width, pipe.height
    ptrs = [ctypes.c_void_p() for _ in range(3)]
    native.check(lib.cw_device_outputs(pipe._h, *[ctypes.byref(q) for q in ptrs]), pipe._h)
    out = []
    for q, nb in zip(ptrs, (w * h * 4, w * h * 4, w * h * 2 * pipe._idx_bytes)):
        buf = np.empty(nb, np.uint8)
        native.check(lib.cw_copy_to_host(pipe._h, buf.ctypes.data, q, nb), pipe._h)
        out.append(buf)
    return out


def _run(params, frames, modes, monkeypatch, chain=True):
    """Push `frames` through one pipeline, frame k by modes[k % len(modes)]
    ("push": cw_push_device on torch's stream, "resident": cw_submit_resident,
    "submit": cw_submit with pinned host frames and outputs); returns the
    per-frame residuals that are observable (host outputs of "submit",
    device outputs after "push") and the final snapshot + device outputs."""
    import torch

    from paper_1408_3526_b200 import Pipeline, _native

    monkeypatch.setenv("CW_CHAIN", "1" if chain else "0")
    monkeypatch.setenv("CW_DYN_STATIC", "1")  # the split chained launches use
    lib = _native.load()
    t, h, w = frames.shape
    dev = torch.from_numpy(frames).cuda()
    host = torch.from_numpy(frames).pin_memory()
    s = torch.cuda.current_stream()
    seen = {}
    with Pipeline(params, w, h) as pipe:
        r, f = ctypes.c_int32(), ctypes.c_int64()
        tickets = []
        outs = {}
        for k in range(t):
            m = modes[k % len(modes)]
            if m == "push":
                while tickets:
                    _native.check(lib.cw_wait(pipe._h, tickets.pop(0), None, None), pipe._h)
                _native.check(lib.cw_push_device(pipe._h, ctypes.c_void_p(dev[k].data_ptr()), ctypes.byref(r),
                                                 ctypes.byref(f), ctypes.c_void_p(s.cuda_stream)), pipe._h)
                torch.cuda.synchronize()
                if r.value:
                    seen[k] = _dev_outputs(lib, pipe, _native)[0].view(np.float32).reshape(h, w).copy()
            else:
                tk = ctypes.c_int64()
                if m == "resident":
                    rc = lib.cw_submit_resident(pipe._h, ctypes.c_void_p(dev[k].data_ptr()), None, None, None,
                                                ctypes.byref(tk))
                else:
                    o = (torch.zeros((h, w), pin_memory=True), torch.zeros((h, w), pin_memory=True),
                         torch.zeros((h, w, 2 * pipe._idx_bytes), dtype=torch.uint8, pin_memory=True))
                    outs[k] = o
                    rc = lib.cw_submit(pipe._h, ctypes.c_void_p(host[k].data_ptr()), ctypes.c_void_p(o[0].data_ptr()),
                                       ctypes.c_void_p(o[1].data_ptr()), ctypes.c_void_p(o[2].data_ptr()),
                                       ctypes.byref(tk))
                _native.check(rc, pipe._h)
                tickets.append((tk.value))
                while len(tickets) > 3:
                    _native.check(lib.cw_wait(pipe._h, tickets.pop(0), None, None), pipe._h)
        while tickets:
            _native.check(lib.cw_wait(pipe._h, tickets.pop(0), None, None), pipe._h)
        torch.cuda.synchronize()
        for k, o in outs.items():
            if k >= params.mz - 1:
                seen[k] = o[0].numpy().copy()
        snap = pipe.snapshot()
        final = _dev_outputs(lib, pipe, _native)
    return seen, snap, final


@pytest.mark.parametrize("shape", [(64, 96), (256, 256), (512, 640)])
def test_resident_chain_matches_serial_launches(params, shape, monkeypatch):
    h, w = shape
    frames = _frames(24, h, w, seed=h)
    _, snap_a, out_a = _run(params, frames, ["push"], monkeypatch, chain=False)
    _, snap_b, out_b = _run(params, frames, ["resident"], monkeypatch, chain=True)
    assert np.array_equal(snap_a, snap_b)
    for x, y in zip(out_a, out_b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("shape", [(64, 96), (512, 640)])
def test_submit_chain_matches_serial_launches(params, shape, monkeypatch):
    """cw_submit with host frames and host outputs (process_stream's call):
    every frame's downloaded residual equals the serialised run's."""
    h, w = shape
    frames = _frames(20, h, w, seed=7)
    seen_a, snap_a, _ = _run(params, frames, ["submit"], monkeypatch, chain=False)
    seen_b, snap_b, _ = _run(params, frames, ["submit"], monkeypatch, chain=True)
    assert np.array_equal(snap_a, snap_b)
    assert sorted(seen_a) == sorted(seen_b) and len(seen_a) >= 10
    for k in seen_a:
        assert np.array_equal(seen_a[k], seen_b[k]), k


def test_mixed_entry_points_match(params, monkeypatch):
    """Chained and plain launches interleaved on one pipeline (a chained
    launch after a plain one, a plain one after a chained one)."""
    frames = _frames(30, 96, 160, seed=11)
    seen_a, snap_a, _ = _run(params, frames, ["push"], monkeypatch, chain=False)
    seen_b, snap_b, _ = _run(params, frames, ["resident", "resident", "submit", "push", "submit", "resident"],
                             monkeypatch, chain=True)
    assert np.array_equal(snap_a, snap_b)
    for k in seen_b:
        assert np.array_equal(seen_a[k], seen_b[k]), k


def test_restore_into_a_chained_stream(params, monkeypatch):
    """Snapshot after 9 frames, restore into a pipeline that already ran a
    chained stream (its flags are ahead of the restored frame count)."""
    import torch

    from paper_1408_3526_b200 import Pipeline, _native

    monkeypatch.setenv("CW_DYN_STATIC", "1")
    frames = _frames(20, 64, 96, seed=3)
    _, snap_ref, out_ref = _run(params, frames, ["submit"], monkeypatch, chain=True)
    lib = _native.load()
    host = torch.from_numpy(frames).pin_memory()
    with Pipeline(params, 96, 64) as a:
        for f in frames[:9]:
            a.process_frame(f)
        snap9 = a.snapshot()
    with Pipeline(params, 96, 64) as b:
        for f in frames[:15]:  # run ahead through the chained submit path
            list(b.process_stream([f]))
        b.restore(snap9)
        for k in range(9, 20):
            tk = ctypes.c_int64()
            o = torch.zeros((64, 96), pin_memory=True)
            _native.check(lib.cw_submit(b._h, ctypes.c_void_p(host[k].data_ptr()), ctypes.c_void_p(o.data_ptr()),
                                        None, None, ctypes.byref(tk)), b._h)
            _native.check(lib.cw_wait(b._h, tk.value, None, None), b._h)
        torch.cuda.synchronize()
        assert np.array_equal(b.snapshot(), snap_ref)


def test_two_chained_pipelines_interleaved(params, monkeypatch):
    """Two pipelines on one GPU, their chained submissions interleaved frame
    by frame: each stream's state equals its own serialised run (the flags
    are per pipeline; a spinning CTA of one never waits on the other)."""
    import torch

    from paper_1408_3526_b200 import Pipeline, _native

    fa = _frames(16, 256, 256, seed=21)
    fb = _frames(16, 96, 160, seed=22)
    _, snap_a, _ = _run(params, fa, ["push"], monkeypatch, chain=False)
    _, snap_b, _ = _run(params, fb, ["push"], monkeypatch, chain=False)
    monkeypatch.setenv("CW_CHAIN", "1")
    lib = _native.load()
    da, db = torch.from_numpy(fa).cuda(), torch.from_numpy(fb).cuda()
    with Pipeline(params, 256, 256) as a, Pipeline(params, 160, 96) as b:
        for k in range(16):
            for pipe, dev in ((a, da), (b, db)):
                tk = ctypes.c_int64()
                _native.check(lib.cw_submit_resident(pipe._h, ctypes.c_void_p(dev[k].data_ptr()), None, None, None,
                                                     ctypes.byref(tk)), pipe._h)
        torch.cuda.synchronize()
        assert np.array_equal(a.snapshot(), snap_a)
        assert np.array_equal(b.snapshot(), snap_b)


def test_process_stream_pageable_frames_chained(params, monkeypatch):
    """process_stream (cw_submit, chained by default) with ordinary pageable
    numpy frames gives the synchronous process_frame results bit for bit
    (static split on both)."""
    from paper_1408_3526_b200 import Pipeline

    monkeypatch.setenv("CW_DYN_STATIC", "1")
    frames = _frames(14, 128, 192, seed=9)
    with Pipeline(params, 192, 128) as p1:
        ref = [p1.process_frame(f) for f in frames]
    with Pipeline(params, 192, 128) as p2:
        got = list(p2.process_stream(list(frames)))
    ref = [r for r in ref if r is not None]
    assert len(ref) == len(got) == 14 - params.mz + 1
    for x, y in zip(ref, got):
        assert x.frame_index == y.frame_index
        assert np.array_equal(x.residual, y.residual)
        assert np.array_equal(x.velocity.indices, y.velocity.indices)


def test_mixed_download_kinds_guard_the_output_sets(params, monkeypatch):
    """Downloads of different kinds two frames apart: a chained cw_submit
    after an event-only (PGM16) download of the same output set, and a
    resident frame after a flagged download -- every downloaded residual
    equals the serialised run's."""
    import torch

    from paper_1408_3526_b200 import Pipeline, _native

    monkeypatch.setenv("CW_DYN_STATIC", "1")
    frames = _frames(24, 64, 96, seed=13)
    q = np.clip(np.rint((frames - 9.0) / 2.0 * 65535.0), 0, 65535).astype(">u2")
    scale, offset = 2.0 / 65535.0, 9.0
    deq = (q.astype(np.float64) * scale + offset).astype(np.float32)
    seen_a, snap_a, _ = _run(params, deq, ["submit"], monkeypatch, chain=False)
    monkeypatch.setenv("CW_CHAIN", "1")
    lib = _native.load()
    dev = torch.from_numpy(deq).cuda()
    host = torch.from_numpy(deq).pin_memory()
    seen = {}
    with Pipeline(params, 96, 64) as pipe:
        tickets, outs = [], {}
        for k in range(24):
            tk = ctypes.c_int64()
            o = torch.zeros((64, 96), pin_memory=True)
            m = ("pgm", "pgm", "f32", "f32", "res", "res")[k % 6]
            if m == "pgm":
                raw = np.ascontiguousarray(q[k])
                rc = lib.cw_submit_raw(pipe._h, raw.ctypes.data, _native.FMT_PGM16, scale, offset,
                                       ctypes.c_void_p(o.data_ptr()), None, None, ctypes.byref(tk))
                outs[k] = (o, raw)
            elif m == "f32":
                rc = lib.cw_submit(pipe._h, ctypes.c_void_p(host[k].data_ptr()), ctypes.c_void_p(o.data_ptr()),
                                   None, None, ctypes.byref(tk))
                outs[k] = (o, None)
            else:
                rc = lib.cw_submit_resident(pipe._h, ctypes.c_void_p(dev[k].data_ptr()), None, None, None,
                                            ctypes.byref(tk))
            _native.check(rc, pipe._h)
            tickets.append(tk.value)
            while len(tickets) > 3:
                _native.check(lib.cw_wait(pipe._h, tickets.pop(0), None, None), pipe._h)
        while tickets:
            _native.check(lib.cw_wait(pipe._h, tickets.pop(0), None, None), pipe._h)
        torch.cuda.synchronize()
        for k, (o, _) in outs.items():
            if k >= params.mz - 1:
                seen[k] = o.numpy().copy()
        assert np.array_equal(pipe.snapshot(), snap_a)
    for k in seen:
        assert np.array_equal(seen[k], seen_a[k]), k


def test_process_resident_matches_process_frame(params, monkeypatch):
    """Pipeline.process_resident (cw_submit_resident with host outputs,
    chained, flagged downloads) gives the synchronous results bit for bit
    (static split on both)."""
    import torch

    from paper_1408_3526_b200 import Pipeline

    monkeypatch.setenv("CW_DYN_STATIC", "1")
    frames = _frames(16, 96, 160, seed=31)
    with Pipeline(params, 160, 96) as p1:
        ref = [o for o in (p1.process_frame(f) for f in frames) if o is not None]
    dev = [torch.from_numpy(f).cuda() for f in frames]
    with Pipeline(params, 160, 96) as p2:
        got = list(p2.process_resident(dev))
    assert len(ref) == len(got) == 16 - params.mz + 1
    for x, y in zip(ref, got):
        assert x.frame_index == y.frame_index
        assert np.array_equal(x.residual, y.residual)
        assert np.array_equal(x.prediction, y.prediction)
        assert np.array_equal(x.velocity.indices, y.velocity.indices)


@pytest.mark.parametrize("mode", ["resident", "submit"])
def test_chain_without_stream_memory_ops(params, mode, monkeypatch):
    """The fallback when cuStreamWriteValue32 is unavailable: resident
    frames copy their ring slot in the kernel prologue, cw_submit waits on
    events; results unchanged."""
    frames = _frames(20, 128, 192, seed=17)
    seen_a, snap_a, _ = _run(params, frames, ["push"] if mode == "resident" else ["submit"], monkeypatch,
                             chain=False)
    monkeypatch.setenv("CW_NO_MEMOPS", "1")
    seen_b, snap_b, _ = _run(params, frames, [mode], monkeypatch, chain=True)
    assert np.array_equal(snap_a, snap_b)
    for k in seen_b:
        assert np.array_equal(seen_a[k], seen_b[k]), k
