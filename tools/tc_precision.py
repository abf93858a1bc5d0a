"""Tensor-core precision study of the lag contraction.

The only GEMM-shaped step of the path is the lag contraction
R^[px, l] = sum_k That[px, k] C[k, l] (K = 162 reals of the smoothed,
kz-collapsed spectrum power, L = 289 lags, pick gains folded into C).  On
tcgen05 it would run with TF32 or BF16 operands (f32 accumulate), or as a
3-pass split ("3xTF32": hi*hi + hi*lo + lo*hi) that recovers ~f32 accuracy.
This script takes the float64 oracle's spectra for a scene, rebuilds the
reference chain in numpy (DC zero, 3-D Hann, power, kz collapse, smoothing;
checked against the oracle's R^), then evaluates the contraction with each
operand precision and reports the velocity-argmax agreement with the
float64 reference on the valid anchors (the parity bar is >= 99.9 % per
frame).  CPU only; the oracle is the checker here, as in tests/.

usage: python tools/tc_precision.py [--size 64] [--frames 32]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import OraclePipeline, autocorr_tables, pick_gains  # noqa: E402
from paper_1408_3526_b200 import default_params  # noqa: E402
from paper_1408_3526_b200.scenegen import SimConfig, generate  # noqa: E402


def round_mantissa(x, bits):
    """Round float64 values to `bits` explicit mantissa bits (nearest even), f32 range."""
    x = np.asarray(x, np.float64).astype(np.float32)
    i = x.view(np.uint32).astype(np.uint64)
    drop = 23 - bits
    half = np.uint64(1 << (drop - 1))
    lsb = (i >> np.uint64(drop)) & np.uint64(1)
    i = (i + half - np.uint64(1) + lsb) & ~np.uint64((1 << drop) - 1)
    return i.astype(np.uint32).view(np.float32).astype(np.float64)


def hann(c, axis):
    return 0.5 * c - 0.25 * np.roll(c, 1, axis=axis) - 0.25 * np.roll(c, -1, axis=axis)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=64)
    ap.add_argument("--frames", type=int, default=32)
    args = ap.parse_args()
    p = default_params()
    kx, ky = p.kx, p.ky
    mx, my, mz = 2 * p.kx + 1, 2 * p.ky + 1, 2 * p.kz + 1
    frames, _ = generate(SimConfig(width=args.size, height=args.size, frame_count=args.frames, rng_seed=0))
    az, axl, ayl = autocorr_tables(p)  # (Mz,), (Lx, Mx), (Ly, My)
    gx, gy = pick_gains(p)
    lx, ly = len(p.lag_grid_x), len(p.lag_grid_y)
    # C[k, (ly, lx)]: R = Re sum_{ky,kx} ayl[ly,ky] axl[lx,kx] T[ky,kx], gains folded
    E = np.einsum("ak,bj->kjab", ayl, axl)  # (My, Mx, Ly, Lx)
    E = E * gy[None, None, :, None] * gx[None, None, None, :]
    C = np.concatenate([E.real.reshape(my * mx, -1), -E.imag.reshape(my * mx, -1)], axis=0)  # (162, 289)
    # pick order: score desc, then |v|^2, ix, iy (the reference's total order)
    vx, vy = np.meshgrid(np.asarray(p.lag_grid_x), np.asarray(p.lag_grid_y))
    order_key = np.lexsort((np.arange(ly)[:, None].repeat(lx, 1).ravel(),
                            np.arange(lx)[None, :].repeat(ly, 0).ravel(), (vx ** 2 + vy ** 2).ravel()))
    rank = np.empty(lx * ly, np.int64)
    rank[order_key] = np.arange(lx * ly)

    def pick(scores):  # (N, 289) -> flat lag index
        best = scores.max(axis=1, keepdims=True)
        cand = np.where(scores == best, rank[None, :], 1 << 30)
        return np.argmin(cand, axis=1)

    modes = {
        "f64": lambda A, B: A @ B,
        "f32 (CUDA cores)": lambda A, B: (A.astype(np.float32) @ B.astype(np.float32)).astype(np.float64),
        "TF32": lambda A, B: round_mantissa(A, 10) @ round_mantissa(B, 10),
        "BF16": lambda A, B: round_mantissa(A, 7) @ round_mantissa(B, 7),
        "3xTF32": lambda A, B: (lambda ah, bh: ah @ bh + ah @ round_mantissa(B - bh, 10)
                                + round_mantissa(A - ah, 10) @ bh)(round_mantissa(A, 10), round_mantissa(B, 10)),
        "3xBF16": lambda A, B: (lambda ah, bh: ah @ bh + ah @ round_mantissa(B - bh, 7)
                                + round_mantissa(A - ah, 7) @ bh)(round_mantissa(A, 7), round_mantissa(B, 7)),
    }
    agree = {m: [] for m in modes}
    margins = []
    that = None
    with OraclePipeline(p, args.size, args.size, threads=os.cpu_count()) as orc:
        for n, f in enumerate(frames):
            out = orc.process_frame(f)
            if out is None:
                continue
            S = orc.sbins()  # (H, W, Mz, My, Mx), k = index - K
            cnd = S.copy()
            cnd[:, :, :, ky, kx] = 0
            for ax in (4, 3, 2):
                cnd = hann(cnd, ax)
            P = cnd.real ** 2 + cnd.imag ** 2
            T = np.einsum("z,hwzyx->hwyx", az, P)
            that = T if that is None else (1 - p.alpha) * T + p.alpha * that
            A = np.concatenate([that.real.reshape(-1, my * mx), that.imag.reshape(-1, my * mx)], axis=1)
            ref = modes["f64"](A, C)
            # the rebuilt chain must reproduce the oracle's R^
            rh = orc.rhat().reshape(-1, ly * lx) * np.outer(gy, gx).ravel()[None, :]
            valid = np.zeros((args.size, args.size), bool)
            valid[my - 1:, mx - 1:] = True
            valid = valid.ravel()
            err = np.abs(ref - rh)[valid].max() / np.abs(rh[valid]).max()
            assert err < 1e-9, f"numpy chain vs oracle R^: {err:.2e}"
            w_ref = pick(ref)
            ix_o = out["indices"][..., 0].ravel()
            iy_o = out["indices"][..., 1].ravel()
            assert np.array_equal((w_ref % lx)[valid], ix_o[valid]) and np.array_equal((w_ref // lx)[valid], iy_o[valid])
            srt = np.sort(ref[valid], axis=1)
            margins.append((srt[:, -1] - srt[:, -2]) / np.abs(srt[:, -1]).clip(1e-300))
            for m, fn in modes.items():
                agree[m].append(np.mean(pick(fn(A, C))[valid] == w_ref[valid]))
    mg = np.concatenate(margins)
    print(f"scene {args.size}x{args.size}x{args.frames} (reference generator, seed 0), "
          f"{len(agree['f64'])} ready frames, {int(valid.sum())} anchors/frame")
    print("relative top-2 score margin quantiles: " + ", ".join(
        f"{q:g}: {np.quantile(mg, q):.2e}" for q in (1e-3, 1e-2, 0.1, 0.5)))
    for m, a in agree.items():
        a = np.asarray(a)
        print(f"{m:18s} min agreement {a.min() * 100:8.4f} %   mean {a.mean() * 100:8.4f} %   "
              f"frames < 99.9 %: {(a < 0.999).sum()}")


if __name__ == "__main__":
    main()
