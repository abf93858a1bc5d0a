"""Frame chaining probe (CW_CHAIN): ms per frame of back-to-back pushes
and the stream state after them, for A/B between processes.

  CW_CHAIN=0|1 python tools/chain_probe.py CONFIG MODE [FRAMES]

MODE: push     -- cw_push_device from a rotating set of device frames
      resident -- cw_submit_resident (chained frame kernels), cw_join for the timing
      submit   -- cw_submit: pinned host frames in, pinned host outputs out, 3 in flight
Prints one JSON line: ms per frame (events around the whole run) and a
sha256 of snapshot() + the last outputs (bit-identity across modes).
"""
import ctypes, hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1408_3526_b200 import FilterParams, Pipeline, _native, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device
from tools.ab_kernel import CONFIGS

cfg = CONFIGS[sys.argv[1]]
mode = sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 400
w, h = cfg["w"], cfg["h"]
p = FilterParams(**cfg["params"]) if cfg["params"] else default_params()
frames = generate_device(SimConfig(width=w, height=h, frame_count=1000), frames=16, nonuniform=cfg.get("nu", False))
lib = _native.load()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
sh = ctypes.c_void_p(s.cuda_stream)
with Pipeline(p, w, h) as pipe:
    r, f = ctypes.c_int32(), ctypes.c_int64()

    tickets = []
    hf = frames.cpu().pin_memory()
    outs = [(torch.empty((h, w), pin_memory=True), torch.empty((h, w), pin_memory=True),
             torch.empty((h, w, 2 * pipe._idx_bytes), dtype=torch.uint8, pin_memory=True)) for _ in range(4)]

    def push(k):
        if mode == "push":
            rc = lib.cw_push_device(pipe._h, ctypes.c_void_p(frames[k % 16].data_ptr()), ctypes.byref(r), ctypes.byref(f), sh)
        else:
            t = ctypes.c_int64()
            if mode == "resident":
                rc = lib.cw_submit_resident(pipe._h, ctypes.c_void_p(frames[k % 16].data_ptr()), None, None, None,
                                            ctypes.byref(t))
            else:
                o = outs[k % 4]
                rc = lib.cw_submit(pipe._h, ctypes.c_void_p(hf[k % 16].data_ptr()), ctypes.c_void_p(o[0].data_ptr()),
                                   ctypes.c_void_p(o[1].data_ptr()), ctypes.c_void_p(o[2].data_ptr()), ctypes.byref(t))
            tickets.append(t.value)
            if len(tickets) > 3:
                _native.check(lib.cw_wait(pipe._h, tickets.pop(0), ctypes.byref(r), ctypes.byref(f)), pipe._h)
        _native.check(rc, pipe._h)

    def drain():
        while tickets:
            _native.check(lib.cw_wait(pipe._h, tickets.pop(0), ctypes.byref(r), ctypes.byref(f)), pipe._h)
        lib.cw_join(pipe._h, sh)

    for k in range(30):
        push(k)
    drain()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for k in range(n):
        push(30 + k)
    if mode != "push":
        lib.cw_join(pipe._h, sh)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    drain()
    torch.cuda.synchronize()
    hs = hashlib.sha256(pipe.snapshot().tobytes())
    ptrs = [ctypes.c_void_p() for _ in range(3)]
    _native.check(lib.cw_device_outputs(pipe._h, *[ctypes.byref(q) for q in ptrs]), pipe._h)
    for q, nb in zip(ptrs, (w * h * 4, w * h * 4, w * h * 2 * pipe._idx_bytes)):
        buf = np.empty(nb, np.uint8)
        _native.check(lib.cw_copy_to_host(pipe._h, buf.ctypes.data, q, nb), pipe._h)
        hs.update(buf.tobytes())
print(json.dumps({"config": sys.argv[1], "mode": mode, "chain": os.environ.get("CW_CHAIN", "0"),
                  "dyn_static": os.environ.get("CW_DYN_STATIC", "default"), "frames": n, "ms_per_frame": ms,
                  "gpx_frames_s": w * h / ms / 1e6, "sha": hs.hexdigest()[:16]}))
