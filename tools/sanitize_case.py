"""Small end-to-end run for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3526_b200 import Pipeline, default_params
rng = np.random.default_rng(0)
frames = (10 + rng.standard_normal((9, 40, 70))).astype(np.float32)
p = default_params()
with Pipeline(p, 70, 40, detect_threshold=0.5) as pipe:
    outs = [o for o in (pipe.process_frame(f) for f in frames) if o is not None]
with Pipeline(p, 70, 40, spectrum_backend="naive") as pipe:
    outs2 = list(pipe.process_stream(frames))
print("ok", len(outs), len(outs2), float(np.abs(outs[-1].residual).max()))
