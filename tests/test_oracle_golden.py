"""Pin the C oracle (oracle/cw_oracle.c) against the REAL reference.

The fixtures in tests/golden/ were produced by the reference package itself
(tests/golden/make_golden.py).  The oracle restates the reference kernels in
the same float64 operation order, so agreement is bit-exact; these tests
are what entitle the GPU parity tests to use the oracle as ground truth.
"""

import numpy as np
import pytest

from conftest import SMALL_CASES, golden, small_case
from oracle.oracle import OraclePipeline, bank_coeffs, retained_bin_indices


def test_oracle_bank_matches_reference_bank(params):
    z = golden("bank_default.npz")
    assert np.array_equal(bank_coeffs(params), z["coeffs"])
    assert np.array_equal(retained_bin_indices(params), z["retained"])


def test_oracle_c1_bit_exact(params):
    z = golden("c1_64x64x32.npz")
    frames = z["frames"]
    y0, y1, x0, x1 = (int(v) for v in z["crop_box"])
    crops = [int(v) for v in z["crop_frames"]]
    k = 0
    with OraclePipeline(params, 64, 64, threads=4) as orc:
        for n in range(frames.shape[0]):
            out = orc.process_frame(frames[n])
            if out is None:
                assert n < params.mz - 1
                continue
            assert out["frame_index"] == z["frame_index"][k]
            assert np.array_equal(out["residual"], z["residual"][k])
            assert np.array_equal(out["prediction"], z["prediction"][k])
            assert np.array_equal(out["indices"], z["indices"][k].astype(np.int32))
            assert out["imag_peak"] == z["imag_peak"][k]
            if n in crops:
                j = crops.index(n)
                assert np.array_equal(orc.sbins()[y0:y1, x0:x1], z["spec_crops"][j])
                assert np.array_equal(orc.rhat()[y0:y1, x0:x1], z["rhat_crops"][j])
            k += 1
    assert k == z["residual"].shape[0] == 28


@pytest.mark.parametrize("name", SMALL_CASES)
def test_oracle_small_cases_bit_exact(name):
    p, frames, forced, outs = small_case(name)
    t, h, w = frames.shape
    k = 0
    with OraclePipeline(p, w, h, threads=3, forced_velocity=forced) as orc:
        for n in range(t):
            out = orc.process_frame(frames[n])
            if out is None:
                continue
            assert np.array_equal(out["residual"], outs["residual"][k])
            assert np.array_equal(out["indices"], outs["indices"][k].astype(np.int32))
            k += 1
    assert k == len(outs["residual"])


def test_oracle_thread_count_invariance(params):
    rng = np.random.default_rng(3)
    frames = rng.random((8, 30, 41)).astype(np.float32)
    outs = []
    for th in (1, 3, 8):
        with OraclePipeline(params, 41, 30, threads=th) as orc:
            outs.append([orc.process_frame(f) for f in frames][-1])
    for o in outs[1:]:
        assert np.array_equal(o["residual"], outs[0]["residual"])
        assert np.array_equal(o["indices"], outs[0]["indices"])
