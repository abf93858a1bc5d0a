"""Golden run of the reference's ``clutterwhiten simulate`` + ``filter`` + ``flow``.

Run in the build container (the reference is importable only there):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_cli_golden.py

Runs the reference CLI (cli.main) exactly as its own test_cli.py does
(32x32, 12 frames, seed 7; filter with --metrics --emit-prediction
--emit-velocity; flow in f32 and csv formats) and stores the input
sequence, ground truth and every output file's content in ``cli_filter.npz``.  tests/test_sequence_gpu.py
replays the input through ``filter_sequence`` and compares file by file.
"""

from __future__ import annotations

import json
import os
import tempfile

import numpy as np

from clutterwhiten.cli import main
from clutterwhiten.seqio import read_sequence

HERE = os.path.dirname(os.path.abspath(__file__))


def main_():
    with tempfile.TemporaryDirectory() as tmp:
        sim, out, met = os.path.join(tmp, "seq"), os.path.join(tmp, "res"), os.path.join(tmp, "m.csv")
        assert main(["simulate", "--out", sim, "--frames", "12", "--seed", "7", "--width", "32",
                     "--height", "32"]) == 0
        assert main(["filter", "--in", sim, "--out", out, "--metrics", met, "--emit-prediction",
                     "--emit-velocity"]) == 0
        flow_f32, flow_csv = os.path.join(tmp, "flow"), os.path.join(tmp, "flowcsv")
        assert main(["flow", "--in", sim, "--out", flow_f32]) == 0
        assert main(["flow", "--in", sim, "--out", flow_csv, "--format", "csv"]) == 0
        flow_meta = json.load(open(os.path.join(flow_f32, "run_meta.json")))
        flow_meta.pop("version", None)
        frames, hin = read_sequence(sim)
        res, hres = read_sequence(out)
        pred, hpred = read_sequence(os.path.join(out, "prediction"))
        vel = np.fromfile(os.path.join(out, "velocity.f32"), dtype="<f4")
        run_meta = json.load(open(os.path.join(out, "run_meta.json")))
        for k in ("seconds", "bank_build_seconds", "version"):
            run_meta.pop(k, None)

        def text(path):
            return np.frombuffer(open(path, "rb").read(), np.uint8)

        np.savez_compressed(
            os.path.join(HERE, "cli_filter.npz"),
            frames=frames, input_header=text(os.path.join(sim, "header.json")),
            ground_truth=text(os.path.join(sim, "ground_truth.json")),
            residual=res, residual_header=np.frombuffer(json.dumps(hres.to_json_dict()).encode(), np.uint8),
            prediction=pred, prediction_header=np.frombuffer(json.dumps(hpred.to_json_dict()).encode(), np.uint8),
            velocity=vel, velocity_json=text(os.path.join(out, "velocity.json")),
            metrics=text(met), run_meta=np.frombuffer(json.dumps(run_meta).encode(), np.uint8),
            flow_velocity=np.fromfile(os.path.join(flow_f32, "velocity.f32"), dtype="<f4"),
            flow_json=text(os.path.join(flow_f32, "velocity.json")),
            flow_csv=text(os.path.join(flow_csv, "velocity.csv")),
            flow_meta=np.frombuffer(json.dumps(flow_meta).encode(), np.uint8))
    print("wrote cli_filter.npz")


if __name__ == "__main__":
    main_()
