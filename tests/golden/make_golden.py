"""Generate the golden fixtures from the REAL reference package.

Run in the build container (the reference is importable only there):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports ``clutterwhiten`` from /root/reference (read-only), runs its own
``Pipeline`` / ``build_bank`` / ``generate`` and stores inputs + outputs as
small .npz fixtures next to this script.  Nothing at test/bench time reads
/root/reference: the fixtures are the committed record of the reference's
behaviour, used to pin the C oracle (tests/test_oracle_golden.py) and the
host layer (tests/test_host_layer.py).
"""

from __future__ import annotations

import os

import numpy as np

import clutterwhiten as cw

HERE = os.path.dirname(os.path.abspath(__file__))


def run(params, frames, forced=None, crops=(), crop_box=None):
    """Run the reference Pipeline; collect every output and optional crops
    of the internal spectrum / smoothed autocorrelation."""
    t, h, w = frames.shape
    out = {"residual": [], "prediction": [], "indices": [], "frame_index": [], "imag_peak": []}
    spec, rhat = [], []
    with cw.Pipeline(params, w, h, forced_velocity=forced) as pipe:
        for n in range(t):
            o = pipe.process_frame(frames[n])
            if o is None:
                continue
            out["residual"].append(o.residual)
            out["prediction"].append(o.prediction)
            out["indices"].append(o.velocity.indices.astype(np.uint8))
            out["frame_index"].append(o.frame_index)
            out["imag_peak"].append(o.imag_peak)
            if n in crops:
                y0, y1, x0, x1 = crop_box
                spec.append(pipe._sbins[y0:y1, x0:x1].copy())
                rhat.append(pipe._rhat[y0:y1, x0:x1].copy())
    res = {k: np.asarray(v) for k, v in out.items()}
    if crops:
        res["spec_crops"] = np.asarray(spec)
        res["rhat_crops"] = np.asarray(rhat)
    return res


def params_dict(p):
    return {
        "kx": p.kx, "ky": p.ky, "kz": p.kz, "bx": p.bx, "by": p.by,
        "mhat": np.asarray(p.mhat), "alpha": p.alpha,
        "lag_grid_x": np.asarray(p.lag_grid_x), "lag_grid_y": np.asarray(p.lag_grid_y),
    }


def main():
    p = cw.default_params()

    # 1. filter bank (design.py:256-274) and retained order (195-205)
    bank = cw.build_bank(p)
    np.savez_compressed(os.path.join(HERE, "bank_default.npz"), coeffs=bank.coeffs, retained=bank.retained)

    # 2. config C1: 64x64x32, reference scene generator, seed 0
    frames, truth = cw.generate(cw.SimConfig(width=64, height=64, frame_count=32, rng_seed=0))
    c1 = run(p, frames, crops=(4, 31), crop_box=(20, 28, 24, 32))
    np.savez_compressed(
        os.path.join(HERE, "c1_64x64x32.npz"), frames=frames, components=truth.components,
        crop_box=np.asarray((20, 28, 24, 32)), crop_frames=np.asarray((4, 31)), **c1,
    )

    # 3. small cases: reference test_pipeline shapes, params sweep
    rng = np.random.default_rng(2026)
    cases = {
        "rand_16x20": (p, rng.random((12, 16, 20)).astype(np.float32), None),
        "const_16x16": (p, np.full((10, 16, 16), 10.0, np.float32), None),
    }
    xs, ys = np.arange(24)[None, :], np.arange(24)[:, None]
    cosine = np.stack([np.cos(2 * np.pi * ((xs - 1.0 * n) / 9 + 2 * (ys - 0.5 * n) / 9)) for n in range(10)])
    cases["forced_cos_24"] = (p, cosine.astype(np.float32), (1.0, 0.5))
    sweep = {
        "k3b2": cw.FilterParams(kx=3, ky=3, kz=2, bx=2, by=2, mhat=(3, 3, 2)),
        "k5b4": cw.FilterParams(kx=5, ky=5, kz=2, bx=4, by=4, mhat=(5, 5, 2)),
        "kz1": cw.FilterParams(kz=1, mhat=(4, 4, 1)),
        "lag_half": cw.FilterParams(lag_grid_x=tuple(i / 2 for i in range(-4, 5)),
                                    lag_grid_y=tuple(i / 2 for i in range(-4, 5))),
        "lag_eighth": cw.FilterParams(lag_grid_x=tuple(i / 8 for i in range(-16, 17)),
                                      lag_grid_y=tuple(i / 8 for i in range(-16, 17))),
    }
    for name, sp in sweep.items():
        fr, _ = cw.generate(cw.SimConfig(width=28, height=26, frame_count=10, rng_seed=5))
        cases[f"sweep_{name}"] = (sp, fr, None)
    blob = {}
    for name, (cp, fr, forced) in cases.items():
        r = run(cp, fr, forced=forced)
        blob[f"{name}/frames"] = fr
        for k, v in r.items():
            blob[f"{name}/{k}"] = v
        for k, v in params_dict(cp).items():
            blob[f"{name}/param_{k}"] = v
        blob[f"{name}/forced"] = np.asarray(forced if forced is not None else (np.nan, np.nan))
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **blob)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
