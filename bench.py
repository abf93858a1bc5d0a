#!/usr/bin/env python
"""Benchmark: pixel-frames/s of the full SDFT -> deadbeat observer -> flow ->
PEF chain on 640x512 frames (BASELINE.json config C3), with % of the HBM
roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one 640x512 frame through the whole per-pixel pipeline (one
fused kernel).  ``value`` is measured with the frames already resident in
HBM (cw_submit_resident: consecutive frame kernels chained, CUDA events on
the kernel stream); ``e2e`` goes through the public
``Pipeline.process_stream`` with pinned host frames (H2D of the frame + D2H
of residual, prediction and velocity per step), and also reports the
synchronous ``Pipeline.process_frame`` rate.
The per-pixel state (1.6 KB/px, 0.5 GB per stream) is larger than L2, so
no L2 flush is needed between steps.  Under torchrun (N > 1) every rank runs
an independent 640x512 sensor stream on its own GPU (streams
shard with no exchange), timed between barriers, max over ranks.
``--gpus N`` without torchrun re-launches this script under
torch.distributed.run with N processes.  The same JSON line carries, under
``c4_strip_sharded``, config C4: one 4096x4096 frame stream split into N
row strips (strips.py), the per-frame NCCL halo exchange inside the timed
region (strong scaling: the total work is fixed).

``--impl reference`` times the reference algorithm on the host cores: the
float64 C restatement in oracle/ (bit-exact to the reference package, see
tests/test_oracle_golden.py), all host threads, same config and metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WIDTH, HEIGHT = 640, 512
METRIC = "pixel-frames/sec (640x512, full pipeline)"
WORKLOAD = "C3: 640x512 frames, full SDFT->deadbeat->autocorr->PEF chain, default FilterParams"
DATA = ("synthetic (reference scene model: 25 drifting cosines + target + counter-based noise, "
        "scenegen.generate_device / generate_counter, seed = rank)")
UNIT = "px-frames/s"
FALLBACK_HBM_GBS = 6650.0


def b_alg(p, with_prediction=True) -> int:
    """Algorithmic HBM bytes per pixel-frame: frame in, delayed
    frame, observer state R+W, smoothing state R+W, residual, velocity pair
    (+ prediction)."""
    return 14 + 8 * (p.mx * p.my * p.mz + p.mx * p.my) + (4 if with_prediction else 0)


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic():
    """dram bytes per launch of the frame kernel from the committed ncu
    capture (profiles/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        if d.get("width") == WIDTH and d.get("height") == HEIGHT:
            return float(d["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.device)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                        rows.append(parts)
        except Exception:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        load = [float(r[1]) for r in rows if float(r[3]) > 250.0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


def dist_setup():
    """(world, rank, CUDA device of this rank).  CW_BENCH_DEVICE pins every
    rank to one device: the multi-rank code path run on a one-GPU box by
    the tests (with CW_BENCH_BACKEND=gloo), never a measurement."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("CW_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    return world, rank, local


def init_dist(local):
    import torch
    import torch.distributed as dist

    backend = os.environ.get("CW_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return dist


def cpu_oracle_rate(params, frames_np, budget_s=12.0, threads=None, max_frames=64):
    """Time the float64 oracle (the reference algorithm) on host cores.
    frames_np: (T, H, W) float32 host frames.  Returns (rate, meta)."""
    from oracle.oracle import OraclePipeline

    threads = threads or os.cpu_count() or 1
    t, h, w = frames_np.shape
    with OraclePipeline(params, w, h, threads=threads) as orc:
        n = 0
        for n in range(params.mz + 1):  # warm-up + one untimed ready frame
            orc.process_frame(frames_np[n % t])
        done, spent = 0, 0.0
        k = params.mz + 1
        while (spent < budget_s or done < 2) and done < max_frames:
            t0 = time.perf_counter()
            orc.process_frame(frames_np[k % t])
            spent += time.perf_counter() - t0
            done += 1
            k += 1
    rate = done * h * w / spent
    return rate, {"cores": threads, "frames": done, "seconds": spent, "height": h, "width": w}


def run_reference(args):
    """--impl reference: the reference algorithm (the float64 C oracle,
    bit-exact to the reference package) on all host cores, on the GPU arm's
    workload -- the same full 640x512 frames (generate_counter, seed 0, bit
    for bit the frames the GPU arm's rank 0 generates on the device), same
    metric.  Each step is one whole frame; the number of timed steps is
    capped so that the run ends within a few minutes."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from paper_1408_3526_b200 import default_params
    from paper_1408_3526_b200.scenegen import SimConfig, generate_counter
    from oracle.oracle import OraclePipeline

    p = default_params()
    threads = os.cpu_count() or 1
    cfg = SimConfig(width=WIDTH, height=HEIGHT, frame_count=1000, rng_seed=0)
    n_frames = min(24, max(8, args.steps + args.warmup + p.mz))  # generated once, cycled
    frames = generate_counter(cfg, frames=n_frames)
    with OraclePipeline(p, WIDTH, HEIGHT, threads=threads) as orc:
        k = 0
        for _ in range(p.mz - 1 + args.warmup):
            orc.process_frame(frames[k % n_frames])
            k += 1
        budget_s = args.ref_budget
        done, dt = 0, 0.0
        while done < args.steps and (dt < budget_s or done < 3):
            t0 = time.perf_counter()
            orc.process_frame(frames[k % n_frames])
            dt += time.perf_counter() - t0
            k += 1
            done += 1
    value = done * HEIGHT * WIDTH / dt
    sample = (f"{done} steady-state 640x512 frames of the C3 scene (of {args.steps} requested; capped at "
              f"{budget_s:.0f} s of CPU time), float64 C oracle = reference algorithm, {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": done, "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / done,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": {"workload": WORKLOAD, "frame": [WIDTH, HEIGHT], "streams": 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import ctypes

    import torch

    from paper_1408_3526_b200 import Pipeline, _native, default_params
    from paper_1408_3526_b200.scenegen import SimConfig, generate_device

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # NCCL's communicator-init log (ranks, transports) for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist = init_dist(local)
    dev = torch.device("cuda", local)
    p = default_params()
    lib = _native.load()

    n_frames = int(min(max(args.steps + args.warmup + p.mz, 64), 1000))
    frames = generate_device(SimConfig(width=WIDTH, height=HEIGHT, frame_count=1000, rng_seed=rank),
                             device=dev, frames=n_frames)
    torch.cuda.synchronize()
    # a dedicated (non-default) stream: the kernels, the frame copies and the
    # timing events all live on it (stream handle 0 would mean "the
    # pipeline's own stream" at the C ABI)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    sh = ctypes.c_void_p(stream.cuda_stream)
    assert sh.value, "expected a non-default CUDA stream"

    pipe = Pipeline(p, WIDTH, HEIGHT, device=local)
    h = pipe._h
    ready, fidx = ctypes.c_int32(), ctypes.c_int64()

    # device-resident frames (generated once, unchanged while in use):
    # cw_submit_resident, whose frame kernels are chained -- each starts in
    # the SM slots the previous frame's early CTAs free
    ticket = ctypes.c_int64()

    def push(k):
        rc = lib.cw_submit_resident(h, ctypes.c_void_p(frames[k % n_frames].data_ptr()), None, None, None,
                                    ctypes.byref(ticket))
        if rc:
            _native.check(rc, h)

    k = 0
    for _ in range(p.mz - 1 + args.warmup):  # fill the temporal window, then warm up
        push(k)
        k += 1
    _native.check(lib.cw_wait(h, ticket.value, ctypes.byref(ready), ctypes.byref(fidx)), h)
    torch.cuda.synchronize()
    assert ready.value == 1
    # no per-launch timing events here: an event with a timestamp between
    # two chained frame kernels serialises them (measured); the stream the
    # kernels run on carries nothing but them, so the timed region's span /
    # steps is the steady-state kernel time per frame
    ms_tot, launches = ctypes.c_double(), ctypes.c_int64()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            push(k)
            k += 1
        _native.check(lib.cw_join(h, sh), h)  # `stream` after the last frame kernel
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    kern_ms = elapsed_ms / args.steps
    launches.value = args.steps
    info = pipe.launch_info()
    pipe.close()

    # ---- e2e through the public API: pinned host frames in, host outputs out ----
    # Pipeline.process_stream: the streaming form of process_frame (every step
    # uploads its frame and downloads residual + prediction + velocity pairs)
    from paper_1408_3526_b200 import Pipeline as PublicPipeline

    e2e_steps = max(args.steps, 300)  # enough frames to amortise the depth-3 pipeline fill
    n_host = min(n_frames, 256)
    host = torch.empty((n_host, HEIGHT, WIDTH), dtype=torch.float32, pin_memory=True)
    host.copy_(frames[:n_host])
    host_np = host.numpy()

    def host_frames(start, count):
        for i in range(count):
            yield host_np[(start + i) % n_host]

    with PublicPipeline(p, WIDTH, HEIGHT, device=local) as pub:
        # warm-up (temporal window + warm-up frames) drained first; then a
        # fresh stream on the warm pipeline: every timed frame is uploaded,
        # processed and downloaded inside the timed region (pipeline fill
        # included, amortised over e2e_steps frames)
        n_pre = p.mz - 1 + args.warmup
        for _ in pub.process_stream(host_frames(0, n_pre)):
            pass
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n_out = 0
        for out in pub.process_stream(host_frames(n_pre, e2e_steps)):
            n_out += 1
        e2e_s = time.perf_counter() - t0
        # the synchronous reference-style call, for the record (warmed up)
        sync_steps = min(e2e_steps, 200)
        for i in range(args.warmup):
            pub.process_frame(host_np[i % n_host])
        t0 = time.perf_counter()
        for i in range(sync_steps):
            out_sync = pub.process_frame(host_np[i % n_host])
        sync_s = time.perf_counter() - t0
        # ... and with ordinary (pageable) numpy frames, as a reference user passes them
        page_np = host_np[: min(n_host, 16)].copy()
        for i in range(args.warmup):
            pub.process_frame(page_np[i % page_np.shape[0]])
        t0 = time.perf_counter()
        for i in range(sync_steps):
            out_sync = pub.process_frame(page_np[i % page_np.shape[0]])
        sync_page_s = time.perf_counter() - t0
    assert n_out == e2e_steps and out_sync is not None
    h2d = WIDTH * HEIGHT * 4
    d2h = WIDTH * HEIGHT * (4 + 4 + 2)

    t = torch.tensor([elapsed_ms, e2e_s, sync_s, sync_page_s], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, e2e_s, sync_s, sync_page_s = (float(v) for v in t)
    px = WIDTH * HEIGHT
    value = world * px * args.steps / (elapsed_ms / 1e3)
    e2e = world * px * e2e_steps / e2e_s
    e2e_sync = world * px * sync_steps / sync_s
    e2e_sync_page = world * px * sync_steps / sync_page_s

    peak, peak_kind = measured_peak()
    bpp = b_alg(p, with_prediction=True)
    achieved = bpp * px / (kern_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(),
                "peak_kind": peak_kind, "bytes_per_px_frame": bpp,
                "kernel_ms": kern_ms, "launches_timed": int(launches.value),
                "kernel_ms_is": ("CUDA-event span of the timed region / launches: the kernel stream carries "
                                 "only the chained frame kernels (consecutive launches overlap), so this is "
                                 "the steady-state kernel time per frame")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        host_frames = frames[: min(n_frames, 16)].cpu().numpy()
        rate, meta = cpu_oracle_rate(p, host_frames, budget_s=args.cpu_budget)
        cpu = {"value": rate, "unit": UNIT, "cores": meta["cores"], "kind": "port",
               "sample": (f"{meta['frames']} steady-state 640x512 C3 frames in {meta['seconds']:.1f}s, "
                          "float64 C oracle (reference algorithm, bit-exact to clutterwhiten)")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": DATA,
            "config": {"workload": WORKLOAD, "frame": [WIDTH, HEIGHT], "streams": world,
                       "parallelism": "independent stream per GPU" if world > 1 else "single GPU",
                       "l2": "state 0.5 GB/stream >> 126 MB L2 (no flush needed)",
                       "grid": info["grid"], "block": info["block"], "smem_bytes": info["smem_bytes"],
                       "api": "cw_submit_resident: device-resident frames, chained frame kernels "
                              "(programmatic dependent launch, per-CTA completion flags)"},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "Pipeline.process_stream (pinned host frames in; host residual, prediction, "
                           "velocity pairs out per step; depth-3 pipelining; every timed frame's upload, "
                           "kernel and download inside the timed region, pipeline fill included)",
                    "steps": e2e_steps,
                    "sync_process_frame": {"value": e2e_sync, "unit": UNIT, "steps": sync_steps,
                                           "frames": "pinned"},
                    "sync_process_frame_pageable": {"value": e2e_sync_page, "unit": UNIT, "steps": sync_steps,
                                                    "frames": "pageable numpy"}},
            "gpu_launches": int(args.steps * info["kernels_per_push"]),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
    c4 = None if args.no_c4 else c4_strip_line(args, lib, dist, world, rank, local, dev)
    if rank == 0:
        line["c4_strip_sharded"] = c4
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def c4_strip_line(args, lib, dist, world, rank, local, dev):
    """Config C4 (BASELINE.json): one 4096x4096 stream split into `world`
    row strips (strips.py); each timed step = this rank's NCCL halo
    exchange (My-1 rows from the rank above) + assembly + the fused kernel
    on its strip.  Device time on a dedicated stream, barriers on both sides,
    max over ranks; value = 4096^2 px per step over that time."""
    import torch

    from paper_1408_3526_b200 import default_params
    from paper_1408_3526_b200.scenegen import SimConfig, generate_device
    from paper_1408_3526_b200.strips import StripPipeline

    w = h = 4096
    p = default_params()
    steps = min(args.steps, args.c4_steps)
    stream = torch.cuda.Stream(device=dev)
    prev = torch.cuda.current_stream(dev)
    torch.cuda.set_stream(stream)
    sp = StripPipeline(p, w, h, rank, world, device=local)
    pl = sp.plan
    own = generate_device(SimConfig(width=w, height=h, frame_count=200, rng_seed=4), device=dev, frames=6,
                          rows=(pl.a0, pl.a1))
    el, kern, n, clk = _device_run(lib, sp.pipe, own, steps, args.warmup, stream, dist, before_push=sp.assemble)
    sp.close()
    del own
    torch.cuda.set_stream(prev)
    t = torch.tensor([el, kern], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    el, kern = float(t[0]), float(t[1])
    peak, peak_kind = measured_peak()
    bpp = b_alg(p)
    rows = pl.a1 - pl.a0  # anchor rows of the largest strip (ranks are equal to +-1 row)
    achieved = bpp * rows * w / (kern / 1e3) / 1e9
    return {
        "metric": "pixel-frames/sec (4096x4096, strip-sharded)", "value": w * h * steps / (el / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": steps, "ms_per_step": el / steps, "scaling": "strong",
        "config": {"workload": "C4: 4096x4096 frames, row strips + (My-1)-row halo exchanged per frame over "
                               + (dist.get_backend().upper() if dist else "nothing (one strip)"),
                   "frame": [w, h], "strips": world, "strip_rows": rows, "halo_rows": p.my - 1 if world > 1 else 0},
        "gpu_launches": steps, "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                                            "frac": achieved / peak, "peak_kind": peak_kind, "kernel_ms": kern,
                                            "bytes_per_px_frame": bpp},
        "clocks": clk,
    }


# ---------------------------------------------------------------------------
# other BASELINE.json configs (extra JSON lines; the driver's default is C3)
# ---------------------------------------------------------------------------

C5_SWEEP = {
    "default (4,4,2,3,3) lag 1/4": dict(),
    "(3,3,2,2,2) lag 1/4": dict(kx=3, ky=3, bx=2, by=2, mhat=(3, 3, 2)),
    "(5,5,2,4,4) lag 1/4": dict(kx=5, ky=5, bx=4, by=4, mhat=(5, 5, 2)),
    "(4,4,1,3,3) lag 1/4": dict(kz=1, mhat=(4, 4, 1)),
    "(4,4,2,3,3) lag 1/2": dict(lag_grid_x=tuple(i / 2 for i in range(-4, 5)),
                                lag_grid_y=tuple(i / 2 for i in range(-4, 5))),
    "(4,4,2,3,3) lag 1/8": dict(lag_grid_x=tuple(i / 8 for i in range(-16, 17)),
                                lag_grid_y=tuple(i / 8 for i in range(-16, 17))),
}


JIT_SWEEP = {
    "(4,4,3,3,3) lag 1/4": dict(kz=3, mhat=(4, 4, 3)),
    "(4,4,2,2,3) lag 1/4": dict(bx=2),
    "(4,3,2,3,2) lag 1/4": dict(ky=3, by=2, mhat=(4, 3, 2)),
}


def _device_run(lib, pipe, frames, steps, warmup, stream, dist=None, before_push=None):
    """Time `steps` device-resident frames (CUDA events, barrier on both
    sides) after the temporal window and `warmup` frames: cw_submit_resident
    (chained frame kernels), or with `before_push` (a frame produced per step
    on `stream`, e.g. the strip assembly) cw_push_device on `stream`; returns
    (elapsed ms, mean kernel ms, launches, clocks summary)."""
    import ctypes

    import torch

    from paper_1408_3526_b200 import _native

    h = pipe._h
    sh = ctypes.c_void_p(stream.cuda_stream)
    ready, fidx = ctypes.c_int32(), ctypes.c_int64()
    nf = frames.shape[0]

    ticket = ctypes.c_int64()

    def push(k):
        if before_push is None:
            rc = lib.cw_submit_resident(h, ctypes.c_void_p(frames[k % nf].data_ptr()), None, None, None,
                                        ctypes.byref(ticket))
        else:
            f = before_push(frames[k % nf])
            rc = lib.cw_push_device(h, ctypes.c_void_p(f.data_ptr()), ctypes.byref(ready), ctypes.byref(fidx), sh)
        if rc:
            _native.check(rc, h)

    k = 0
    for _ in range(pipe.params.mz - 1 + warmup):
        push(k)
        k += 1
    torch.cuda.synchronize()
    timed = before_push is not None  # per-launch events (they would serialise chained launches)
    if timed:
        lib.cw_set_timing(h, 1)
    ms_tot, launches = ctypes.c_double(), ctypes.c_int64()
    lib.cw_kernel_time(h, ctypes.byref(ms_tot), ctypes.byref(launches))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clocks:
        ev0.record(stream)
        for _ in range(steps):
            push(k)
            k += 1
        lib.cw_join(h, sh)
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    el = ev0.elapsed_time(ev1)
    if not timed:
        return el, el / steps, steps, clocks.summary()
    lib.cw_kernel_time(h, ctypes.byref(ms_tot), ctypes.byref(launches))
    lib.cw_set_timing(h, 0)
    return el, ms_tot.value / max(1, launches.value), int(launches.value), clocks.summary()


def run_config(args):
    """--config c2 | c4 | c5: the other BASELINE.json configurations."""
    import torch

    from paper_1408_3526_b200 import FilterParams, Pipeline, _native, default_params
    from paper_1408_3526_b200.scenegen import SimConfig, generate_device

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist = init_dist(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    lib = _native.load()
    peak, peak_kind = measured_peak()
    lines = []

    def maxrank(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def line(metric, workload, px_per_step, p, elapsed, kern, launches, clocks, scaling, extra):
        ms = maxrank(elapsed)
        d = {"metric": metric, "value": px_per_step * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
             "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
             "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
             "data": "synthetic (reference scene model, generated on device)",
             "config": dict(workload=workload, **extra), "gpu_launches": args.steps,
             "roofline": {"bound": "hbm", "achieved": b_alg(p) * px_per_step / world / (kern / 1e3) / 1e9,
                          "peak": peak, "unit": "GB/s", "peak_kind": peak_kind,
                          "frac": b_alg(p) * px_per_step / world / (kern / 1e3) / 1e9 / peak,
                          "traffic": None, "bytes_per_px_frame": b_alg(p), "kernel_ms": kern,
                          "launches_timed": launches},
             "clocks": clocks}
        lines.append(d)

    if args.config == "c2":
        w = h = 256
        p = default_params()
        frames = generate_device(SimConfig(width=w, height=h, frame_count=256, rng_seed=2 + rank), device=dev,
                                 nonuniform=True)
        with Pipeline(p, w, h, device=local) as pipe:
            el, kern, n, clk = _device_run(lib, pipe, frames, args.steps, args.warmup, stream, dist)
        line("pixel-frames/sec (256x256, non-uniform motion)", "C2: 256x256x256, non-uniform background motion",
             w * h * world, p, el, kern, n, clk, "weak", {"frame": [w, h], "streams": world})
    elif args.config == "c5":
        w, h = 1280, 1024
        frames = generate_device(SimConfig(width=w, height=h, frame_count=1000, rng_seed=rank), device=dev,
                                 frames=16)
        for name, kw in C5_SWEEP.items():
            p = FilterParams(**kw)
            with Pipeline(p, w, h, device=local) as pipe:
                el, kern, n, clk = _device_run(lib, pipe, frames, args.steps, args.warmup, stream, dist)
            line("pixel-frames/sec (1280x1024 stream per GPU, params sweep)", f"C5: {name}", w * h * world, p, el,
                 kern, n, clk, "weak", {"frame": [w, h], "streams": world, "params": name})
    elif args.config == "jit":
        # legal geometries with no instance in the library: the
        # fused kernel compiled at run time (NVRTC) vs the runtime-geometry
        # kernels, 1280x1024
        w, h = 1280, 1024
        frames = generate_device(SimConfig(width=w, height=h, frame_count=1000, rng_seed=rank), device=dev,
                                 frames=16)
        for name, kw in JIT_SWEEP.items():
            p = FilterParams(**kw)
            for path in ("fused (run-time compiled)", "runtime-geometry kernels"):
                if path.startswith("runtime"):
                    os.environ["CW_NO_JIT"] = "1"
                with Pipeline(p, w, h, device=local) as pipe:
                    kind = int(lib.cw_kernel_kind(pipe._h))
                    steps = args.steps if kind != 2 else max(3, min(args.steps, 30))
                    el, kern, n, clk = _device_run(lib, pipe, frames, steps, args.warmup, stream, dist)
                os.environ.pop("CW_NO_JIT", None)
                line("pixel-frames/sec (1280x1024, geometry without a compiled instance)", f"{name}: {path}",
                     w * h * world, p, el * args.steps / steps, kern, n, clk, "weak",
                     {"frame": [w, h], "params": name, "kernel_kind": kind})
    elif args.config == "c3naive":
        # the paper's naive-vs-recursive comparison at 640x512
        p = default_params()
        frames = generate_device(SimConfig(width=WIDTH, height=HEIGHT, frame_count=1000, rng_seed=rank),
                                 device=dev, frames=32)
        for backend in ("recursive", "naive"):
            with Pipeline(p, WIDTH, HEIGHT, device=local, spectrum_backend=backend) as pipe:
                el, kern, n, clk = _device_run(lib, pipe, frames, args.steps, args.warmup, stream, dist)
            line("pixel-frames/sec (640x512, full pipeline)", f"C3 with spectrum_backend={backend}",
                 WIDTH * HEIGHT * world, p, el, kern, n, clk, "weak",
                 {"frame": [WIDTH, HEIGHT], "spectrum_backend": backend})
    elif args.config == "c3seq":
        # stored sequence -> fused kernel -> stored residuals
        # (filter_sequence: reader thread, 3 frames in flight, writer thread);
        # wall clock of the whole file-to-file run, pipeline setup excluded
        from paper_1408_3526_b200.seqio import SequenceWriter
        from paper_1408_3526_b200.sequence import filter_sequence

        p = default_params()
        n_frames = min(max(args.steps, 64), 600)  # pgm16 output buffers frames for its global range
        src = generate_device(SimConfig(width=WIDTH, height=HEIGHT, frame_count=1000, rng_seed=rank), device=dev,
                              frames=32).cpu().numpy()
        with tempfile.TemporaryDirectory(prefix="cw_seq_") as tmp:
            for fmt in ("f32le", "pgm16"):
                with SequenceWriter(os.path.join(tmp, fmt), WIDTH, HEIGHT, dtype=fmt) as wr:
                    for t in range(n_frames):
                        wr.append(src[t % 32])
                meta = filter_sequence(os.path.join(tmp, fmt), os.path.join(tmp, fmt + "_out"), p, device=local,
                                       metrics=os.path.join(tmp, fmt + ".csv"))
                ms = meta["seconds"] * 1e3
                lines.append({
                    "metric": "pixel-frames/sec (640x512, sequence file -> residual file + metrics)",
                    "value": WIDTH * HEIGHT * n_frames / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": n_frames,
                    "warmup": 0, "ms_per_step": ms / n_frames, "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference scene model)",
                    "config": {"workload": f"C3 frames stored as {fmt}; filter_sequence to f32le residuals",
                               "input_format": fmt, "frames": n_frames, "frame": [WIDTH, HEIGHT],
                               "storage": tmp},
                    "wall_clock": True})
    elif args.config == "c4":
        from paper_1408_3526_b200.strips import StripPipeline

        w = h = 4096
        p = default_params()
        sp = StripPipeline(p, w, h, rank, world, device=local)
        pl = sp.plan
        own = generate_device(SimConfig(width=w, height=h, frame_count=200, rng_seed=4), device=dev, frames=6,
                              rows=(pl.a0, pl.a1))
        el, kern, n, clk = _device_run(lib, sp.pipe, own, args.steps, args.warmup, stream, dist,
                                       before_push=sp.assemble)
        sp.close()
        line("pixel-frames/sec (4096x4096, strip-sharded)", "C4: 4096x4096, row strips + 8-row halo over NCCL",
             w * h, p, el, kern, n, clk, "strong", {"frame": [w, h], "strips": world, "halo_rows": p.my - 1})
    elif args.config == "c4strips":
        # C4 strip decomposition measured on ONE GPU (this environment has no
        # multi-GPU box): for N = 1, 2, 4, 8 the kernel runs the strip a rank
        # of an N-way split owns (the middle one, with its My-1 halo rows) and
        # the line reports the projected N-GPU rate 4096^2 / strip time.  The
        # per-frame halo exchange (8 rows x 4096 x 4 B = 128 KiB from one
        # neighbour over NVLink) is not in the timed region.
        from paper_1408_3526_b200.strips import plan_strips

        w = h = 4096
        p = default_params()
        for n_strips in (1, 2, 4, 8):
            pl = plan_strips(p, h, n_strips)[n_strips // 2]
            frames = generate_device(SimConfig(width=w, height=h, frame_count=200, rng_seed=4), device=dev,
                                     frames=6, rows=(pl.lo, pl.a1))
            with Pipeline(p, w, pl.local_height, device=local, _strip=(pl.halo, pl.lo)) as pipe:
                el, kern, n, clk = _device_run(lib, pipe, frames, args.steps, args.warmup, stream, dist)
            line("pixel-frames/sec (4096x4096, strip-sharded), projected from one strip on 1 GPU",
                 f"C4: strip {n_strips // 2} of {n_strips} (rows {pl.lo}..{pl.a1}, halo {pl.halo}) timed alone",
                 w * h, p, el, kern, n, clk, "strong",
                 {"frame": [w, h], "strips": n_strips, "strip_rows": pl.a1 - pl.a0, "halo_rows": pl.halo,
                  "projection": "N-GPU rate = 4096^2 / (one strip's time); halo exchange excluded"})
            # roofline of the strip kernel: algorithmic bytes of the strip's own anchor rows
            lines[-1]["roofline"]["achieved"] *= (pl.a1 - pl.a0) / h
            lines[-1]["roofline"]["frac"] *= (pl.a1 - pl.a0) / h
    if rank == 0:
        for d in lines:
            print(json.dumps(d), flush=True)
    if dist:
        dist.destroy_process_group()


def relaunch(n: int) -> int:
    """`--gpus N` outside torchrun: run this script again as N ranks, one per
    GPU (torch.distributed.run, 127.0.0.1), NCCL's init log enabled."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU-oracle timing")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 strip-sharded block of the headline line")
    ap.add_argument("--c4-steps", type=int, default=400, help="timed frames of the C4 block (capped by --steps)")
    ap.add_argument("--ref-budget", type=float, default=60.0,
                    help="--impl reference: seconds of timed CPU work (steps are capped to fit)")
    ap.add_argument("--config", choices=("c3", "c2", "c4", "c4strips", "c5", "c3naive", "c3seq", "jit"), default="c3",
                    help="c3 (default, the headline) or another BASELINE.json configuration")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    elif args.config != "c3":
        run_config(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
