"""Break down Pipeline.process_frame time at 640x512 (host side)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1408_3526_b200 import Pipeline, _native, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device

W, H = 640, 512
fr = generate_device(SimConfig(width=W, height=H, frame_count=1000), frames=64)
pinned = torch.empty((64, H, W), dtype=torch.float32, pin_memory=True); pinned.copy_(fr)
pin_np = pinned.numpy()
page_np = fr.cpu().numpy()
p = default_params()
lib = _native.load()
def timeit(fn, n=100):
    for _ in range(5): fn()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    return (time.perf_counter() - t0) / n * 1e3
with Pipeline(p, W, H) as pipe:
    for k in range(8): pipe.process_frame(pin_np[k])
    k = [8]
    def full_pinned():
        pipe.process_frame(pin_np[k[0] % 64]); k[0] += 1
    def full_page():
        pipe.process_frame(page_np[k[0] % 64]); k[0] += 1
    res = np.empty((H, W), np.float32); pred = np.empty_like(res); vidx = np.empty((H, W, 2), np.uint8)
    pres = torch.empty((H, W), dtype=torch.float32, pin_memory=True).numpy(); ppred = torch.empty((H, W), dtype=torch.float32, pin_memory=True).numpy()
    pvidx = torch.empty((H, W, 2), dtype=torch.uint8, pin_memory=True).numpy()
    r, f = ctypes.c_int32(), ctypes.c_int64()
    def raw(res=res, pred=pred, vidx=vidx):
        lib.cw_push(pipe._h, _native.fptr(pin_np[k[0] % 64]), _native.fptr(res), _native.fptr(pred),
                    vidx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), ctypes.byref(r), ctypes.byref(f), None); k[0] += 1
    def raw_pinned_out(): raw(pres, ppred, pvidx)
    def raw_nores():
        lib.cw_push(pipe._h, _native.fptr(pin_np[k[0] % 64]), None, None, None, ctypes.byref(r), ctypes.byref(f), None); k[0] += 1
        torch.cuda.synchronize()
    def wrap(): pipe._wrap(0, res, pred, vidx)
    def alloc(): np.empty((H, W), np.float32); np.empty((H, W), np.float32); np.empty((H, W, 2), np.uint8)
    for name, fn in [("process_frame pinned in", full_pinned), ("process_frame pageable in", full_page),
                     ("cw_push pinned in, pageable out", raw), ("cw_push pinned in, pinned out", raw_pinned_out),
                     ("cw_push no outputs (H2D+kernel)", raw_nores), ("_wrap (astype + lag lookup)", wrap), ("3x np.empty", alloc)]:
        print(f"{name:40s} {timeit(fn):8.3f} ms")
