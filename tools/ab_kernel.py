"""A/B kernel timing of several builds of the library on one GPU.

  python tools/ab_kernel.py [--frames N] [--rounds R] [--config c3|c2|c5lag8|c5k5] lib1.so lib2.so ...

A library argument may carry environment settings for its runs:
``lib.so@CW_DYN_STATIC=0.8,CW_DYN_CHUNK=4``.

Each (round, lib) runs in its own process (the library is loaded once per
process): N device-resident frames through cw_push_device, CUDA events
around every frame kernel (cw_set_timing), mean kernel ms.  Rounds
alternate the libraries so that clock / power drift hits all of them.
"""

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import ctypes, json, os, sys
sys.path.insert(0, {root!r})
import torch
from paper_1408_3526_b200 import FilterParams, Pipeline, _native, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device
cfg = {cfg!r}
n = {n}
w, h, kw = cfg["w"], cfg["h"], cfg["params"]
p = FilterParams(**kw) if kw else default_params()
frames = generate_device(SimConfig(width=w, height=h, frame_count=1000), frames=16, nonuniform=cfg.get("nu", False))
lib = _native.load()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
with Pipeline(p, w, h) as pipe:
    r, f = ctypes.c_int32(), ctypes.c_int64()
    sh = ctypes.c_void_p(s.cuda_stream)
    def push(k):
        _native.check(lib.cw_push_device(pipe._h, ctypes.c_void_p(frames[k % 16].data_ptr()), ctypes.byref(r), ctypes.byref(f), sh), pipe._h)
    for k in range(30):
        push(k)
    torch.cuda.synchronize()
    lib.cw_set_timing(pipe._h, 1)
    ms, cnt = ctypes.c_double(), ctypes.c_int64()
    lib.cw_kernel_time(pipe._h, ctypes.byref(ms), ctypes.byref(cnt))
    for k in range(n):
        push(30 + k)
    torch.cuda.synchronize()
    lib.cw_kernel_time(pipe._h, ctypes.byref(ms), ctypes.byref(cnt))
print(json.dumps({{"kernel_ms": ms.value / cnt.value}}))
"""

CONFIGS = {
    "c3": {"w": 640, "h": 512, "params": {}},
    "c2": {"w": 256, "h": 256, "params": {}, "nu": True},
    "c5": {"w": 1280, "h": 1024, "params": {}},
    "c5lag8": {"w": 1280, "h": 1024, "params": {"lag_grid_x": tuple(i / 8 for i in range(-16, 17)),
                                                 "lag_grid_y": tuple(i / 8 for i in range(-16, 17))}},
    "c5lag2": {"w": 1280, "h": 1024, "params": {"lag_grid_x": tuple(i / 2 for i in range(-4, 5)),
                                                 "lag_grid_y": tuple(i / 2 for i in range(-4, 5))}},
    "c5k5": {"w": 1280, "h": 1024, "params": {"kx": 5, "ky": 5, "bx": 4, "by": 4, "mhat": (5, 5, 2)}},
    "c5k3": {"w": 1280, "h": 1024, "params": {"kx": 3, "ky": 3, "bx": 2, "by": 2, "mhat": (3, 3, 2)}},
    "c5kz1": {"w": 1280, "h": 1024, "params": {"kz": 1, "mhat": (4, 4, 1)}},
    "jit433": {"w": 1280, "h": 1024, "params": {"kz": 3, "mhat": (4, 4, 3)}},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=2000)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    res = {lib: [] for lib in a.libs}
    code = CHILD.format(root=ROOT, cfg=cfg, n=a.frames)
    for _ in range(a.rounds):
        for lib in a.libs:
            path, _, extra = lib.partition("@")
            env = dict(os.environ, CW_B200_LIB=os.path.abspath(path))
            for kv in filter(None, extra.split(",")):
                k, _, v = kv.partition("=")
                env[k] = v
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            try:
                res[lib].append(json.loads(out.stdout.strip().splitlines()[-1])["kernel_ms"])
            except Exception:
                print(lib, "failed:", out.stderr[-800:], flush=True)
    px = cfg["w"] * cfg["h"]
    for lib, v in res.items():
        if v:
            v = sorted(v)
            print(f"{a.config} {os.path.basename(lib):48s} kernel_ms min {v[0]:.5f} median {v[len(v) // 2]:.5f} "
                  f"({px / v[len(v) // 2] / 1e6:.3f} Gpx-frames/s) all {['%.5f' % x for x in v]}", flush=True)


if __name__ == "__main__":
    main()
