"""Per-warp phase clocks of CTA 0 (needs libcw_b200_timing.so built with
-DCW_PHASE_TIMING); 640x512 frames, averaged per row."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["CW_B200_LIB"] = os.path.join(ROOT, "paper_1408_3526_b200", os.environ.get("CW_TIMING_LIB", "libcw_b200_timing.so"))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1408_3526_b200 import Pipeline, _native, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device
W, H = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (640, 512)
fr = generate_device(SimConfig(width=W, height=H, frame_count=1000), frames=16)
lib = _native.load()
lib.cw_phase_clocks.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * (128 + 2048))()
names = ["tail F/loop", "xstage+ySDFT", "TMA wait", "observer+Hz+Hx", "bar1", "C1 Hy/pow/T", "bar2", "CD contract", "bar3", "E pick+PEF", "bar4"]
with Pipeline(default_params(), W, H) as pipe:
    r, f = ctypes.c_int32(), ctypes.c_int64()
    for k in range(10):
        lib.cw_push_device(pipe._h, ctypes.c_void_p(fr[k % 16].data_ptr()), ctypes.byref(r), ctypes.byref(f), None)
    torch.cuda.synchronize()
    lib.cw_phase_clocks(buf)  # discard warm-up
    n = 20
    for k in range(n):
        lib.cw_push_device(pipe._h, ctypes.c_void_p(fr[k % 16].data_ptr()), ctypes.byref(r), ctypes.byref(f), None)
    torch.cuda.synchronize()
    lib.cw_phase_clocks(buf)
    grid = pipe.launch_info()["grid"]
a = np.array(buf[:128], dtype=np.float64).reshape(8, 16)[:5, :11]
rows = (W // 32) * H / grid  # rows per CTA per frame
a = a / (n * rows)
print(f"cycles per row (CTA 0, {rows:.1f} rows/frame), warps 0..4:")
for i, nm in enumerate(names):
    print(f"  {nm:16s}" + "".join(f"{a[w, i]:9.0f}" for w in range(5)))
print(f"  {'total':16s}" + "".join(f"{a[w].sum():9.0f}" for w in range(5)))

# per-CTA spans of the last launch (globaltimer ns)
sp = np.array(buf[128:], dtype=np.float64).reshape(1024, 2)[:grid]
t0 = sp[:, 0].min()
st, en = (sp[:, 0] - t0) / 1e3, (sp[:, 1] - t0) / 1e3
print(f"CTA spans (us, last launch, {grid} CTAs): start max {st.max():.2f}; end min {en.min():.2f} "
      f"p50 {np.median(en):.2f} p90 {np.percentile(en, 90):.2f} max {en.max():.2f}; duration p50 {np.median(en - st):.2f}")
