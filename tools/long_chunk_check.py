"""Recursive vs naive spectrum backend on tall frames (long CTA runs): velocity agreement and residual error per frame."""
import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from paper_1408_3526_b200 import Pipeline, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device
from parity import velocity_agreement, agreeing_outputs, residual_error
p = default_params(); w, h = 1280, 2048
frames = generate_device(SimConfig(width=w, height=h, frame_count=200, rng_seed=3), frames=8).cpu().numpy()
outs = {}
for backend in ("recursive", "naive"):
    with Pipeline(p, w, h, spectrum_backend=backend) as pipe:
        outs[backend] = [o for o in (pipe.process_frame(f) for f in frames) if o is not None]
fmax = float(np.abs(frames).max())
for a, b in zip(outs["recursive"], outs["naive"]):
    va = velocity_agreement(a.velocity.indices, b.velocity.indices.astype(np.int32), p)
    m = a.mask & agreeing_outputs(a.velocity.indices, b.velocity.indices, p)
    print(os.environ.get("CW_B200_LIB","intree")[-14:], f"vel {va:.6f} res {residual_error(a.residual, b.residual, m, fmax):.2e}")
