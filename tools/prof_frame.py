"""Short 640x512 run for ncu: N frames through the fused kernel."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1408_3526_b200 import Pipeline, _native, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
w, h = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (640, 512)
frames = generate_device(SimConfig(width=w, height=h, frame_count=1000), device="cuda", frames=16)
lib = _native.load()
p = default_params()
with Pipeline(p, w, h) as pipe:
    r, f = ctypes.c_int32(), ctypes.c_int64()
    for k in range(n):
        _native.check(lib.cw_push_device(pipe._h, ctypes.c_void_p(frames[k % 16].data_ptr()), ctypes.byref(r), ctypes.byref(f), None), pipe._h)
    torch.cuda.synchronize()
print("ok", n, "frames")
