"""Sequence-storage fixtures written and read by the REAL reference seqio.

Run in the build container (the reference is importable only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_seq_golden.py

Writes tests/golden/seq/<case>/ directories with the reference's
``write_sequence`` (f32le and pgm16, default and explicit quantisation), one
hand-made PGM16 header with comments / odd whitespace that the reference's
reader accepts, and ``seq_expected.npz`` holding the reference's
``read_sequence`` result for every case.  tests/test_seqio.py checks that
our writer reproduces these bytes and our reader (host and GPU decode)
reproduces these values.
"""

from __future__ import annotations

import json
import os
import shutil

import numpy as np

from clutterwhiten.seqio import read_sequence, write_sequence

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "seq")


def main():
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    rng = np.random.default_rng(1408)
    cases = {}
    f32 = (rng.standard_normal((3, 5, 7)) * 40).astype(np.float32)
    write_sequence(f32, os.path.join(OUT, "f32le"), meta={"seed": 1408})
    cases["f32le"] = dict(frames=f32)
    signed = (rng.standard_normal((4, 9, 11)) * 3 - 1).astype(np.float32)
    write_sequence(signed, os.path.join(OUT, "pgm16_signed"), dtype="pgm16")
    cases["pgm16_signed"] = dict(frames=signed)
    write_sequence(np.full((2, 4, 4), -3.5, np.float32), os.path.join(OUT, "pgm16_const"), dtype="pgm16")
    cases["pgm16_const"] = {}
    scene = (10.0 + rng.standard_normal((3, 6, 8))).astype(np.float32)
    write_sequence(scene, os.path.join(OUT, "pgm16_fixed"), dtype="pgm16", scale=1.0 / 512, offset=4.0,
                   meta={"source": "fixture"})
    cases["pgm16_fixed"] = dict(frames=scene)
    # a PGM with comments and mixed whitespace in its header
    d = os.path.join(OUT, "pgm16_comments")
    os.makedirs(d)
    q = rng.integers(0, 65536, size=(3, 5), dtype=np.uint16)
    with open(os.path.join(d, "frame_000000.pgm"), "wb") as fh:
        fh.write(b"P5 # sensor A\n# exposure 1ms\n5\t3\r\n65535\n" + q.astype(">u2").tobytes())
    with open(os.path.join(d, "header.json"), "w") as fh:
        json.dump({"width": 5, "height": 3, "frame_count": 1, "dtype": "pgm16",
                   "scale": 0.001, "offset": -7.25, "meta": {}}, fh)
    cases["pgm16_comments"] = {}

    expected = {}
    for name in cases:
        frames, hdr = read_sequence(os.path.join(OUT, name))
        expected[f"{name}__read"] = frames
        expected[f"{name}__header"] = np.frombuffer(json.dumps(hdr.to_json_dict()).encode(), np.uint8)
        if "frames" in cases[name]:
            expected[f"{name}__written"] = cases[name]["frames"]
    # metrics rows of cli.compute_metrics_row on synthetic outputs, with and
    # without ground truth (ties in |res| exercise the first-in-row-major rule)
    from clutterwhiten.cli import compute_metrics_row
    from clutterwhiten.flow import VelocityField
    from clutterwhiten.params import default_params
    from clutterwhiten.pipeline import WhitenedOutput, valid_mask
    from clutterwhiten.scenegen import GroundTruth, SimConfig

    params = default_params()
    h, w = 24, 20
    mask = valid_mask(params, w, h)
    res = (rng.standard_normal((3, h, w)) * 0.1).astype(np.float32)
    res[1, 10, 7] = res[1, 12, 9] = -0.75  # tie: first in row-major order wins
    res *= mask
    idx = rng.integers(0, 17, size=(3, h, w, 2)).astype(np.int32)
    lag = np.asarray(params.lag_grid_x)
    cfg = SimConfig(width=w, height=h, frame_count=6)
    centers = np.array([[9.5 + 0.25 * t, 11.0 - 0.5 * t] for t in range(6)])
    truth = GroundTruth(config=cfg, seed=0, components=np.zeros((0, 4)), clutter_velocity=(1.625, 0.625),
                        target_centers=centers)
    rows_nt, rows_t = [], []
    for k in range(3):
        vel = VelocityField(indices=idx[k], velocities=np.stack([lag[idx[k, ..., 0]], lag[idx[k, ..., 1]]], -1))
        out = WhitenedOutput(frame_index=2 + k, residual=res[k], prediction=np.zeros_like(res[k]), velocity=vel,
                             mask=mask, imag_peak=0.0)
        rows_nt.append(compute_metrics_row(out, params, None).csv())
        rows_t.append(compute_metrics_row(out, params, truth).csv())
    expected["metrics__residual"] = res
    expected["metrics__indices"] = idx
    expected["metrics__truth"] = np.frombuffer(json.dumps(truth.to_json_dict()).encode(), np.uint8)
    expected["metrics__rows_no_truth"] = np.array(rows_nt)
    expected["metrics__rows_truth"] = np.array(rows_t)
    np.savez_compressed(os.path.join(HERE, "seq_expected.npz"), **expected)
    print("wrote", sorted(cases))


if __name__ == "__main__":
    main()
