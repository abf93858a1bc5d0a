"""Per-warp phase clocks of CTA 0 and per-CTA spans (needs a library built
with -DCW_PHASE_TIMING, e.g. tools/dev_build.sh build/libcw_timing.so
-DCW_PHASE_TIMING; CW_TIMING_LIB names it relative to the package dir).

  python tools/phase_timing.py [W H] [--resident]

--resident pushes the frames through cw_submit_resident (chained frame
kernels) and also prints, for the last two frames, how long each CTA
waited for its predecessor and the gap between a CTA's end and its
successor's start."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["CW_B200_LIB"] = os.path.join(ROOT, "paper_1408_3526_b200", os.environ.get("CW_TIMING_LIB", "libcw_b200_timing.so"))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1408_3526_b200 import Pipeline, _native, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device
args = [a for a in sys.argv[1:] if not a.startswith("--")]
resident = "--resident" in sys.argv
W, H = (int(args[0]), int(args[1])) if len(args) > 1 else (640, 512)
fr = generate_device(SimConfig(width=W, height=H, frame_count=1000), frames=16)
lib = _native.load()
lib.cw_phase_clocks.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * (128 + 12288))()
names = ["tail F/loop", "xstage+ySDFT", "TMA wait", "observer+Hz+Hx", "bar1", "C1 Hy/pow/T", "bar2", "CD contract", "bar3", "E pick+PEF", "bar4"]
with Pipeline(default_params(), W, H) as pipe:
    r, f = ctypes.c_int32(), ctypes.c_int64()
    t = ctypes.c_int64()

    def push(k):
        if resident:
            lib.cw_submit_resident(pipe._h, ctypes.c_void_p(fr[k % 16].data_ptr()), None, None, None, ctypes.byref(t))
        else:
            lib.cw_push_device(pipe._h, ctypes.c_void_p(fr[k % 16].data_ptr()), ctypes.byref(r), ctypes.byref(f), None)

    for k in range(10):
        push(k)
    torch.cuda.synchronize()
    lib.cw_phase_clocks(buf)  # discard warm-up
    n = 40
    for k in range(n):
        push(k)
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

# per-CTA spans of the last two launches (globaltimer ns): [seq & 1][CTA]
# [start, setup, ring copy, pre-roll, chain wait, end]
sp = np.array(buf[128:], dtype=np.float64).reshape(2, 1024, 6)[:, :grid][:, :, [0, 1, 2, 3, 4, 5]]
last = int(np.argmax(sp[:, :, 5].max(axis=1)))  # the parity of the later launch
cur, prev = sp[last], sp[1 - last]
t0 = cur[:, 0].min()
st, en = (cur[:, 0] - t0) / 1e3, (cur[:, 5] - t0) / 1e3
print(f"CTA spans (us, last launch, {grid} CTAs): start max {st.max():.2f}; end min {en.min():.2f} "
      f"p50 {np.median(en):.2f} p90 {np.percentile(en, 90):.2f} max {en.max():.2f}; duration p50 {np.median(en - st):.2f}")
if resident:
    dur = (cur[:, 5] - cur[:, 0]) / 1e3
    wait = (cur[:, 4] - cur[:, 0]) / 1e3
    gap = (cur[:, 0] - prev[:, 5]) / 1e3  # successor start - predecessor end (negative: started before it ended)
    period = (cur[:, 5].max() - prev[:, 5].max()) / 1e3
    d = np.diff(cur[:, :5], axis=1) / 1e3
    print("prologue (us, mean / p90): " + ", ".join(
        f"{nm} {d[:, i].mean():.2f} / {np.percentile(d[:, i], 90):.2f}"
        for i, nm in enumerate(["setup", "ring copy", "pre-roll", "chain wait"])))
    print(f"chained: frame period (last end to last end) {period:.2f} us; CTA duration mean {dur.mean():.2f} "
          f"p50 {np.median(dur):.2f}; waited for the predecessor mean {wait.mean():.2f} p90 {np.percentile(wait, 90):.2f}; "
          f"start - predecessor end mean {gap.mean():.2f} min {gap.min():.2f} max {gap.max():.2f}; "
          f"work after the wait mean {(dur - wait).mean():.2f}")
