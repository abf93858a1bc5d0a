"""Host layer (CPU): parameters, bank design, scene generator and the
Pipeline's pre-device checks, against the reference's behaviour
(golden fixtures from tests/golden/make_golden.py) and its own tests'
known answers (test_params.py, test_design.py, test_pipeline.py)."""

import math
import os

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_1408_3526_b200 import (
    ExecStrategy, FilterParams, ParamError, Pipeline, build_bank, default_params, dirichlet,
    kernel_to_freq, load_params, pick_gains, retained_bin_indices, sample_kernel, save_params,
    valid_bounds, valid_mask, validate,
)
from paper_1408_3526_b200._native import NativeUnavailable
from paper_1408_3526_b200.pipeline import apply_pef
from paper_1408_3526_b200.scenegen import SimConfig, generate


# -- params (params.py:34-251) ------------------------------------------------

def test_default_derived_sizes(params):
    assert (params.mx, params.my, params.mz) == (9, 9, 5)
    assert (params.wx, params.wy) == (7, 7)
    assert params.bin_count == 405 and params.retained_count == 245
    assert params.latency == 2 and params.delta == (4, 4, 2)
    assert params.alpha == pytest.approx(math.exp(-0.1))
    assert len(params.lag_grid_x) == 17 and params.lag_grid_x[0] == -2.0


@pytest.mark.parametrize("kw, match", [
    (dict(kx=0), "half-window"),
    (dict(bx=4), "B < K"),
    (dict(by=-1), "B < K"),
    (dict(mhat=(9, 4, 2)), "group delay"),
    (dict(mhat=(4, 4)), "3 components"),
    (dict(alpha=1.0), "smoothing pole"),
    (dict(lag_grid_x=()), "must not be empty"),
    (dict(lag_grid_x=(0.0, 0.0)), "strictly increasing"),
    (dict(lag_grid_y=(0.0, float("nan"))), "non-finite"),
    (dict(lag_grid_x=(-4.5, 0.0)), "span exceeds"),
    (dict(kx=2.0), "must be an integer"),
])
def test_validate_rejects(kw, match):
    with pytest.raises(ParamError, match=match):
        validate(FilterParams(**kw))


def test_params_file_round_trip(tmp_path):
    p = FilterParams(kx=3, ky=3, bx=2, by=2, mhat=(3, 3, 2), lag_grid_x=(-1.0, 0.0, 1.0))
    f = tmp_path / "p.txt"
    save_params(p, f)
    assert load_params(f) == p


def test_params_file_errors(tmp_path):
    f = tmp_path / "bad.txt"
    f.write_text("kx = 4\nbogus = 1\n")
    with pytest.raises(ParamError, match="unknown parameter key"):
        load_params(f)
    f.write_text("kx = 4\nkx = 3\n")
    with pytest.raises(ParamError, match="duplicate key"):
        load_params(f)
    f.write_text("kx = four\n")
    with pytest.raises(ParamError, match="bad value"):
        load_params(f)


# -- design (design.py) ---------------------------------------------------------

def test_bank_matches_reference_golden(params, default_bank):
    z = golden("bank_default.npz")
    assert default_bank.coeffs.shape == z["coeffs"].shape == (17, 17, 5, 7, 7)
    assert np.abs(default_bank.coeffs - z["coeffs"]).max() < 1e-7
    assert np.array_equal(default_bank.retained, z["retained"])
    assert np.array_equal(retained_bin_indices(params), z["retained"])


def test_bank_matches_per_velocity_design_path(params, default_bank):
    for ix, iy in ((0, 0), (8, 8), (3, 14), (16, 5)):
        vx, vy = params.lag_grid_x[ix], params.lag_grid_y[iy]
        ref = kernel_to_freq(sample_kernel(params, (vx, vy)), params).coeffs
        assert np.abs(default_bank.coeffs[iy, ix] - ref).max() < 1e-7


def test_dirichlet_known_answers():
    assert dirichlet(0.0, 7) == 1.0
    assert dirichlet(3.0, 7) == 1.0
    assert dirichlet(0.5, 3) == pytest.approx(-1.0 / 3.0)
    with pytest.raises(ValueError):
        dirichlet(0.1, 4)


def test_tap_sum_unit_and_centre_tap(params):
    for v in ((0.0, 0.0), (1.25, -0.5), (-2.0, 2.0)):
        assert abs(sample_kernel(params, v).taps.sum() - 1.0) < 1e-10
    assert sample_kernel(params, (0.0, 0.0)).taps[2, 4, 4] == pytest.approx(49 / 405)


def test_bank_index_of(default_bank):
    assert default_bank.index_of((0.0, 0.0)) == (8, 8)
    with pytest.raises(ParamError, match="not on the configured velocity grid"):
        default_bank.index_of((0.3, 0.0))


def test_pick_gains_unit_at_zero_lag(params):
    gx, gy = pick_gains(params)
    assert gx[8] == pytest.approx(1.0) and gy[8] == pytest.approx(1.0)
    assert np.all(gx >= 1.0)


# -- pipeline helpers and pre-device checks (pipeline.py) -------------------------

def test_valid_region_defaults(params):
    assert valid_bounds(params, 64, 64) == (4, 59, 4, 59)
    m = valid_mask(params, 64, 64)
    assert m.sum() == 56 * 56 and m[4, 4] and m[59, 59] and not m[3, 10]


def test_apply_pef_matches_direct_convolution(params, default_bank):
    rng = np.random.default_rng(50)
    mx, my, mz = np.arange(9), np.arange(9), np.arange(5)
    kx, ky, kz = mx - 4, my - 4, mz - 2
    phase = (kz[:, None, None, None, None, None] * mz[None, None, None, :, None, None] / 5
             + ky[None, :, None, None, None, None] * my[None, None, None, None, :, None] / 9
             + kx[None, None, :, None, None, None] * mx[None, None, None, None, None, :] / 9)
    basis = (np.exp(2j * np.pi * phase) / np.sqrt(405)).reshape(405, 405)
    for _ in range(10):
        window = rng.random((5, 9, 9))
        ix, iy = (int(v) for v in rng.integers(0, 17, 2))
        kern = default_bank.kernel(ix, iy)
        bins = (basis @ window.ravel()).reshape(5, 9, 9)
        pred, res = apply_pef(bins, kern, 1.0)
        direct = float(np.sum(sample_kernel(params, kern.velocity).taps * window))
        assert abs(pred - direct) <= 1e-4 * window.max()
        assert res == pytest.approx(1.0 - pred)


def test_strategy_parsing():
    assert ExecStrategy.parse("serial").name == "serial"
    assert ExecStrategy.parse("parallel:3").workers == 3
    with pytest.raises(ValueError, match="workers >= 1"):
        ExecStrategy.parse("parallel:0")
    with pytest.raises(ValueError):
        ExecStrategy.parse("threads")


def test_pipeline_rejects_before_touching_the_device(params, default_bank):
    with pytest.raises(ParamError):
        Pipeline(params, 4, 4, bank=default_bank)
    with pytest.raises(ParamError, match="different parameters"):
        Pipeline(FilterParams(alpha=0.5), 16, 16, bank=default_bank)
    with pytest.raises(ParamError):
        Pipeline(params, 16, 16, bank=default_bank, forced_velocity=(0.3, 0.0))
    with pytest.raises(ValueError, match="unknown spectrum backend"):
        Pipeline(params, 16, 16, bank=default_bank, spectrum_backend="fft")
    with pytest.raises(ValueError, match="workers >= 1"):
        Pipeline(params, 16, 16, bank=default_bank, strategy="parallel:0")


def test_no_cpu_fallback_without_a_gpu(params, default_bank):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(NativeUnavailable):
        Pipeline(params, 16, 16, bank=default_bank)


# -- scene generator (scenegen.py) ------------------------------------------------

def test_scene_generator_reproduces_reference_bits():
    z = golden("c1_64x64x32.npz")
    frames, comps = generate(SimConfig(width=64, height=64, frame_count=32, rng_seed=0))
    assert np.array_equal(comps, z["components"])
    assert np.array_equal(frames, z["frames"])


def test_product_package_never_touches_the_oracle():
    """The float64 oracle is test infrastructure: no module of the product
    package imports, loads or names it (static check of the sources)."""
    import ast
    import os

    import paper_1408_3526_b200 as pkg

    root = os.path.dirname(pkg.__file__)
    for name in sorted(os.listdir(root)):
        if not name.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(root, name)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert not any(a.name.split(".")[0] == "oracle" for a in node.names), name
            elif isinstance(node, ast.ImportFrom):
                assert (node.module or "").split(".")[0] != "oracle", name
            elif isinstance(node, ast.Constant) and isinstance(node.value, str):
                assert "libcw_oracle" not in node.value, name


def test_reference_arm_line_on_cpu():
    """bench.py --impl reference (the reference algorithm = the float64 oracle
    on the host cores): same metric, workload and unit as the GPU arm, with
    the cpu_baseline / e2e objects the contract asks for."""
    import json
    import subprocess
    import sys

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3", "--ref-budget", "0.5"], capture_output=True, text=True, cwd=ROOT,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    import bench

    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["config"]["workload"] == bench.WORKLOAD and d["config"]["frame"] == [640, 512]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
