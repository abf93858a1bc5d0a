"""Sequence storage and metrics rows vs the reference (CPU).

Pinned to fixtures written / read / scored by the reference itself
(tests/golden/make_seq_golden.py): our writer must reproduce its bytes, our
reader its values, our metrics rows its CSV text.  The remaining cases
restate the reference's own test_seqio.py (/root/reference/pkg/tests/
test_seqio.py:14-129).
"""

import json
import os

import numpy as np
import pytest

from paper_1408_3526_b200 import default_params
from paper_1408_3526_b200.pipeline import valid_mask
from paper_1408_3526_b200.seqio import (SequenceError, SequenceHeader, SequenceReader, SequenceWriter,
                                        read_sequence, write_sequence)
from paper_1408_3526_b200.sequence import (METRICS_HEADER, GroundTruthLite, load_ground_truth, metrics_row)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SEQ = os.path.join(GOLD, "seq")
EXP = np.load(os.path.join(GOLD, "seq_expected.npz"))
CASES = ["f32le", "pgm16_signed", "pgm16_const", "pgm16_fixed", "pgm16_comments"]


def _hdr(name):
    return json.loads(EXP[f"{name}__header"].tobytes().decode())


def _files(d):
    return {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))}


@pytest.mark.parametrize("name", CASES)
def test_reader_matches_reference(name):
    frames, hdr = read_sequence(os.path.join(SEQ, name))
    want = EXP[f"{name}__read"]
    assert frames.dtype == np.float32 and frames.shape == want.shape
    assert np.array_equal(frames.view(np.uint32), want.view(np.uint32))
    assert hdr.to_json_dict() == _hdr(name)


@pytest.mark.parametrize("name,kw", [("f32le", dict(meta={"seed": 1408})),
                                     ("pgm16_signed", dict(dtype="pgm16")),
                                     ("pgm16_fixed", dict(dtype="pgm16", scale=1.0 / 512, offset=4.0,
                                                          meta={"source": "fixture"}))])
def test_writer_reproduces_reference_bytes(tmp_path, name, kw):
    write_sequence(EXP[f"{name}__written"], tmp_path / "s", **kw)
    assert _files(tmp_path / "s") == _files(os.path.join(SEQ, name))


@pytest.mark.parametrize("dtype", ["f32le", "pgm16"])
def test_streaming_writer_equals_bulk(tmp_path, dtype):
    frames = EXP["pgm16_signed__written"]
    write_sequence(frames, tmp_path / "bulk", dtype=dtype, meta={"k": 1})
    with SequenceWriter(tmp_path / "stream", frames.shape[2], frames.shape[1], dtype=dtype, meta={"k": 1}) as wr:
        for f in frames:
            wr.append(f)
    assert _files(tmp_path / "stream") == _files(tmp_path / "bulk")


@pytest.mark.parametrize("name", CASES)
def test_raw_payload_and_frame_reads(name):
    want = EXP[f"{name}__read"]
    with SequenceReader(os.path.join(SEQ, name)) as rd:
        assert len(rd) == want.shape[0] and rd.shape == want.shape[1:]
        for t in range(len(rd)):
            assert np.array_equal(rd.read(t), want[t])
            raw = np.empty(want.shape[1:], dtype=rd.raw_dtype)
            rd.read_raw(t, raw)
            if not rd.pgm:
                assert np.array_equal(raw.astype(np.float32), want[t])
            else:
                h = rd.header
                assert np.array_equal((raw.astype(np.float64) * h.scale + h.offset).astype(np.float32), want[t])


# --- the reference's own seqio cases (test_seqio.py) -------------------------

def test_f32_round_trip_bit_identical(tmp_path):
    frames = (np.random.default_rng(1).standard_normal((7, 12, 10)) * 40).astype(np.float32)
    hdr = write_sequence(frames, tmp_path / "seq", meta={"seed": 1})
    back, hdr2 = read_sequence(tmp_path / "seq")
    assert np.array_equal(back, frames)
    assert (hdr2.width, hdr2.height, hdr2.frame_count, hdr2.dtype, hdr2.meta) == (10, 12, 7, "f32le", {"seed": 1})
    assert hdr.to_json_dict() == hdr2.to_json_dict()


def test_pgm16_round_trip_within_quantization(tmp_path):
    frames = (np.random.default_rng(2).standard_normal((4, 9, 11)) * 3 - 1).astype(np.float32)
    write_sequence(frames, tmp_path / "seq", dtype="pgm16")
    back, hdr = read_sequence(tmp_path / "seq")
    step = (float(frames.max()) - float(frames.min())) / 65535.0
    assert np.abs(back.astype(np.float64) - frames).max() <= step
    assert hdr.scale == pytest.approx(step) and back.min() < 0


def test_pgm16_constant_sequence(tmp_path):
    write_sequence(np.full((2, 4, 4), -3.5, dtype=np.float32), tmp_path / "seq", dtype="pgm16")
    back, hdr = read_sequence(tmp_path / "seq")
    assert np.allclose(back, -3.5) and hdr.scale == 1.0


def test_pgm_payload_is_big_endian_p5(tmp_path):
    write_sequence(np.array([[[0.0, 1.0]]], dtype=np.float32), tmp_path / "seq", dtype="pgm16")
    header, payload = (tmp_path / "seq" / "frame_000000.pgm").read_bytes().split(b"65535\n", 1)
    assert header.startswith(b"P5\n2 1\n") and payload == b"\x00\x00\xff\xff"


def test_truncated_payloads_rejected(tmp_path):
    write_sequence(np.zeros((3, 4, 4), dtype=np.float32), tmp_path / "a")
    raw = tmp_path / "a" / "frames.f32"
    raw.write_bytes(raw.read_bytes()[:-8])
    with pytest.raises(SequenceError, match="expected"):
        read_sequence(tmp_path / "a")
    write_sequence(np.zeros((1, 4, 4), dtype=np.float32), tmp_path / "b", dtype="pgm16")
    p = tmp_path / "b" / "frame_000000.pgm"
    p.write_bytes(p.read_bytes()[:-2])
    with pytest.raises(SequenceError, match="truncated"):
        read_sequence(tmp_path / "b")


def test_malformed_and_missing_header_rejected(tmp_path):
    write_sequence(np.zeros((1, 4, 4), dtype=np.float32), tmp_path / "seq")
    (tmp_path / "seq" / "header.json").write_text("{not json")
    with pytest.raises(SequenceError, match="malformed"):
        read_sequence(tmp_path / "seq")
    (tmp_path / "seq" / "header.json").write_text(json.dumps({"width": 4}))
    with pytest.raises(SequenceError, match="malformed"):
        read_sequence(tmp_path / "seq")
    (tmp_path / "empty").mkdir()
    with pytest.raises(SequenceError, match="missing header.json"):
        read_sequence(tmp_path / "empty")


def test_header_validation_and_bad_shapes(tmp_path):
    with pytest.raises(SequenceError, match="dtype"):
        SequenceHeader(4, 4, 1, dtype="f64").validate()
    with pytest.raises(SequenceError, match="scale"):
        SequenceHeader(4, 4, 1, scale=0.0).validate()
    with pytest.raises(SequenceError):
        write_sequence(np.zeros((4, 4), dtype=np.float32), tmp_path / "x")
    with pytest.raises(SequenceError):
        write_sequence(np.zeros((1, 4, 4), dtype=np.float32), tmp_path / "y", dtype="png8")


def test_header_dimension_mismatch_with_pgm(tmp_path):
    write_sequence(np.zeros((1, 4, 6), dtype=np.float32), tmp_path / "seq", dtype="pgm16")
    hp = tmp_path / "seq" / "header.json"
    data = json.loads(hp.read_text())
    data["width"] = 5
    hp.write_text(json.dumps(data))
    with pytest.raises(SequenceError, match="header says"):
        read_sequence(tmp_path / "seq")


# --- metrics rows vs cli.compute_metrics_row ---------------------------------

class _Vel:
    def __init__(self, v):
        self.velocities = v


class _O:
    def __init__(self, fidx, res, mask, vel, metrics=None):
        self.frame_index, self.residual, self.mask, self.velocity, self.metrics = fidx, res, mask, vel, metrics


def _metric_inputs():
    p = default_params()
    res, idx = EXP["metrics__residual"], EXP["metrics__indices"]
    mask = valid_mask(p, res.shape[2], res.shape[1])
    lag = np.asarray(p.lag_grid_x)
    return p, res, idx, mask, lag


def test_metrics_rows_match_reference(tmp_path):
    p, res, idx, mask, lag = _metric_inputs()
    (tmp_path / "ground_truth.json").write_bytes(EXP["metrics__truth"].tobytes())
    truth = load_ground_truth(tmp_path)
    assert isinstance(truth, GroundTruthLite)
    for k in range(res.shape[0]):
        vel = _Vel(np.stack([lag[idx[k, ..., 0]], lag[idx[k, ..., 1]]], -1))
        o = _O(2 + k, res[k], mask, vel)
        assert metrics_row(o, p, None).csv() == str(EXP["metrics__rows_no_truth"][k])
        assert metrics_row(o, p, truth).csv() == str(EXP["metrics__rows_truth"][k])
    assert METRICS_HEADER.count(",") == 9


def test_metrics_row_from_fused_stats():
    """The no-truth row built from the kernel epilogue's (peak, sum of f64
    squares, count) equals the host computation when those stats are exact."""
    p, res, idx, mask, lag = _metric_inputs()
    for k in range(res.shape[0]):
        r = res[k]
        a = np.where(mask, np.abs(r), -1.0)
        flat = int(np.argmax(a))
        st = {"peak_abs_residual": float(np.abs(r).flat[flat]), "peak_x": flat % r.shape[1],
              "peak_y": flat // r.shape[1], "sum_sq": float(np.sum(r[mask].astype(np.float64) ** 2)),
              "n_valid": int(mask.sum())}
        row = metrics_row(_O(2 + k, r, mask, None, st), p, None)
        assert row.csv() == str(EXP["metrics__rows_no_truth"][k])


def test_writer_reproduces_reference_cli_input(tmp_path):
    """The input sequence of the reference CLI golden run (make_cli_golden.py)
    re-written by our writer: identical header and payload bytes."""
    g = np.load(os.path.join(GOLD, "cli_filter.npz"))
    hdr = g["input_header"].tobytes().decode()
    write_sequence(g["frames"], tmp_path / "s", meta=json.loads(hdr)["meta"])
    assert (tmp_path / "s" / "header.json").read_text() == hdr
    back, _ = read_sequence(tmp_path / "s")
    assert np.array_equal(back, g["frames"])
