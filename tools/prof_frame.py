"""Short run for ncu: N frames through the fused kernel.

  python tools/prof_frame.py [N] [config]     config: a tools/ab_kernel.py CONFIGS key (default c3)
  python tools/prof_frame.py N W H            (default parameters on a W x H frame)
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1408_3526_b200 import FilterParams, Pipeline, _native, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device
from tools.ab_kernel import CONFIGS

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
if len(sys.argv) > 3:
    cfg = {"w": int(sys.argv[2]), "h": int(sys.argv[3]), "params": {}}
else:
    cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c3"]
w, h = cfg["w"], cfg["h"]
p = FilterParams(**cfg["params"]) if cfg["params"] else default_params()
frames = generate_device(SimConfig(width=w, height=h, frame_count=1000), device="cuda", frames=16,
                         nonuniform=cfg.get("nu", False))
lib = _native.load()
with Pipeline(p, w, h) as pipe:
    r, f = ctypes.c_int32(), ctypes.c_int64()
    for k in range(n):
        _native.check(lib.cw_push_device(pipe._h, ctypes.c_void_p(frames[k % 16].data_ptr()), ctypes.byref(r), ctypes.byref(f), None), pipe._h)
    torch.cuda.synchronize()
print("ok", n, "frames", w, h)
