"""Parity metrics (stated tolerances).

* velocity: fraction of valid anchors whose (ix, iy) equals the oracle's
  (target >= 0.999 per frame)
* residual: max |res - res_ref| over valid outputs <= 1e-4 * max|I|
* spectrum: per pixel max_k |S - S_ref| / max_k |S_ref| <= 1e-5
* R^: per pixel max_l |R - R_ref| / max_l |R_ref| <= 1e-5
The reference's per-bin relative metric (bench.py:175-182) is not used: it
is ill-conditioned at near-zero bins and unattainable in float32.
"""

import numpy as np

VEL_FRAC = 0.999
RES_TOL = 1e-4
SPEC_TOL = 1e-5
RHAT_TOL = 1e-5


def anchor_mask(params, h, w, y_off=0):
    m = np.zeros((h, w), bool)
    m[max(0, params.my - 1 - y_off):, params.mx - 1:] = True
    return m


def velocity_agreement(idx, idx_ref, params):
    h, w = idx.shape[:2]
    m = anchor_mask(params, h, w)
    same = np.all(idx == idx_ref, axis=-1)
    return float(same[m].mean())


def residual_error(res, res_ref, mask, frames_max):
    return float(np.abs(res[mask].astype(np.float64) - res_ref[mask]).max() / frames_max)


def per_pixel_rel(a, b, axes):
    num = np.abs(a - b).max(axis=axes)
    den = np.abs(b).max(axis=axes)
    ok = den > 0
    out = np.zeros_like(num)
    out[ok] = num[ok] / den[ok]
    out[~ok] = num[~ok]
    return float(out.max())


def agreeing_outputs(idx, idx_ref, params):
    """Output pixels (anchor - mhat) whose anchor picked the same velocity."""
    mhx, mhy, _ = params.mhat
    same = np.all(idx == idx_ref, axis=-1)
    h, w = same.shape
    out = np.zeros((h, w), bool)
    out[: h - mhy, : w - mhx] = same[mhy:, mhx:]
    return out
