"""Print parity diagnostics (GPU vs golden/oracle) for C1."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import golden
from paper_1408_3526_b200 import Pipeline, default_params
from paper_1408_3526_b200.pipeline import rhat_from_state
from parity import per_pixel_rel

p = default_params()
z = golden("c1_64x64x32.npz")
frames = z["frames"]
fmax = np.abs(frames).max()
y0, y1, x0, x1 = (int(v) for v in z["crop_box"])
with Pipeline(p, 64, 64) as pipe:
    k = 0
    for n in range(32):
        o = pipe.process_frame(frames[n])
        if o is None:
            continue
        idx = o.velocity.indices
        ref = z["indices"][k].astype(np.int32)
        same = np.all(idx == ref, axis=-1)
        sa = same[8:, 8:]
        agree_out = np.zeros((64, 64), bool)
        agree_out[:60, :60] = same[4:, 4:]
        d = np.abs(o.residual.astype(np.float64) - z["residual"][k])
        m = o.mask & agree_out
        print(f"n={n} fi={o.frame_index} vel_agree={sa.mean():.5f} flips={(~sa).sum()} "
              f"res_err_agree={d[m].max()/fmax:.3e} res_err_all={d[o.mask].max()/fmax:.3e} "
              f"pred_err={np.abs(o.prediction-z['prediction'][k])[m].max():.3e}")
        if n in (4, 31):
            j = (4, 31).index(n)
            s = pipe.spectrum()[y0:y1, x0:x1]
            print("   spec rel", per_pixel_rel(s, z["spec_crops"][j], axes=(-3, -2, -1)))
            rh = rhat_from_state(pipe.smoothed_state()[y0:y1, x0:x1], p)
            print("   rhat rel", per_pixel_rel(rh, z["rhat_crops"][j], axes=(-2, -1)))
        if (~sa).sum() > 0 and n < 12:
            ys, xs = np.nonzero(~sa)
            for yy, xx in list(zip(ys, xs))[:3]:
                print("    flip at", yy + 8, xx + 8, idx[yy+8, xx+8], ref[yy+8, xx+8])
        k += 1
