"""bench.py's driver contract (one JSON line with the required keys) at
N = 1 and through the multi-rank code path.  The N = 2 run pins both ranks
to cuda:0 over gloo (CW_BENCH_DEVICE / CW_BENCH_BACKEND) to exercise the
re-launch under torch.distributed.run, the barriers, the max over ranks
and the strip-sharded C4 block with its halo exchange; it checks the code
path, it is not a measurement (the ranks share one GPU)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks")


def _run(args, env=None, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         env=dict(os.environ, **(env or {})), timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_one_gpu_contract():
    d = _run(["--steps", "40", "--warmup", "3", "--no-cpu-baseline", "--c4-steps", "5"])
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 40 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 640 * 512 * 4
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.2
    assert d["gpu_launches"] == 40
    c4 = d["c4_strip_sharded"]
    assert c4["n_gpus"] == 1 and c4["config"]["strips"] == 1 and c4["value"] > 0


@pytest.mark.gpu
def test_bench_multi_rank_code_path():
    d = _run(["--gpus", "2", "--steps", "20", "--warmup", "3", "--no-cpu-baseline", "--c4-steps", "5"],
             env={"CW_BENCH_BACKEND": "gloo", "CW_BENCH_DEVICE": "0"})
    assert d["n_gpus"] == 2 and d["config"]["streams"] == 2
    assert d["config"]["parallelism"] == "independent stream per GPU"
    c4 = d["c4_strip_sharded"]
    assert c4["n_gpus"] == 2 and c4["config"]["strips"] == 2 and c4["config"]["halo_rows"] == 8
    assert "GLOO" in c4["config"]["workload"] and c4["value"] > 0
