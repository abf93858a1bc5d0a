"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything
else runs on a CPU-only host (the driver runs ``-m "not gpu"`` here)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def small_case(name):
    """(params, frames, forced, outputs) of one golden small case."""
    from paper_1408_3526_b200 import FilterParams

    z = golden("small_cases.npz")
    g = lambda k: z[f"{name}/{k}"]
    p = FilterParams(
        kx=int(g("param_kx")), ky=int(g("param_ky")), kz=int(g("param_kz")),
        bx=int(g("param_bx")), by=int(g("param_by")),
        mhat=tuple(int(v) for v in g("param_mhat")), alpha=float(g("param_alpha")),
        lag_grid_x=tuple(float(v) for v in g("param_lag_grid_x")),
        lag_grid_y=tuple(float(v) for v in g("param_lag_grid_y")),
    )
    forced = g("forced")
    forced = None if np.isnan(forced).any() else (float(forced[0]), float(forced[1]))
    outs = {k: g(k) for k in ("residual", "prediction", "indices", "frame_index", "imag_peak")}
    return p, g("frames"), forced, outs


SMALL_CASES = (
    "rand_16x20", "const_16x16", "forced_cos_24",
    "sweep_k3b2", "sweep_k5b4", "sweep_kz1", "sweep_lag_half", "sweep_lag_eighth",
)


@pytest.fixture(scope="session")
def params():
    from paper_1408_3526_b200 import default_params

    return default_params()


@pytest.fixture(scope="session")
def default_bank(params):
    from paper_1408_3526_b200 import build_bank

    return build_bank(params)
