"""KLRM snapshots and CSV import on the host (reference
tests/test_matrixio.py: round trip, header layout, corruption, CSV cap).
CPU only; the streaming device reader is covered in test_gpu_matrixio.py."""

import struct

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st
from hypothesis.extra import numpy as hnp

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import matrixio as mio
from paper_2104_10785_b200 import synth


def test_bits_survive(tmp_path):
    A = synth.gaussian_matrix(13, 7, seed=2)
    p = tmp_path / "a.klrm"
    K.write_matrix(p, A)
    B = K.read_matrix(p)
    assert B.dtype == np.float64 and np.array_equal(A, B)


@settings(max_examples=40, deadline=None)
@given(hnp.arrays(np.float64, hnp.array_shapes(min_dims=2, max_dims=2, min_side=1, max_side=6),
                  elements=st.floats(-1e12, 1e12)))
def test_roundtrip_property(A):
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        K.write_matrix(f"{d}/m.klrm", A)
        assert np.array_equal(K.read_matrix(f"{d}/m.klrm"), A)


def test_header_layout(tmp_path):
    A = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    p = tmp_path / "h.klrm"
    K.write_matrix(p, A)
    raw = p.read_bytes()
    magic, ver, rows, cols = struct.unpack("<4sIQQ", raw[:24])
    assert (magic, ver, rows, cols) == (b"KLRM", 1, 3, 2)
    assert raw[24:] == A.tobytes(order="C")


def test_noncontiguous_and_f32_inputs_are_stored_as_f64(tmp_path):
    A = synth.gaussian_matrix(9, 8, seed=3)
    p = tmp_path / "s.klrm"
    K.write_matrix(p, A[::2, 1:].astype(np.float32))
    B = K.read_matrix(p)
    assert B.dtype == np.float64 and np.array_equal(B, A[::2, 1:].astype(np.float32))


def test_rejects_non_2d(tmp_path):
    with pytest.raises(K.ShapeMismatchError):
        K.write_matrix(tmp_path / "v.klrm", np.ones(4))


def _corrupt(tmp_path, edit):
    p = tmp_path / "x.klrm"
    K.write_matrix(p, np.eye(3))
    bad = tmp_path / "bad.klrm"
    bad.write_bytes(edit(p.read_bytes()))
    return bad


@pytest.mark.parametrize("edit,msg", [
    (lambda r: b"NOPE" + r[4:], "bad magic"),
    (lambda r: r[:4] + struct.pack("<I", 99) + r[8:], "unsupported format version 99"),
    (lambda r: r[:-8], "payload holds 64 bytes, header promises 72"),
    (lambda r: b"KLRM\x01", "truncated header"),
])
def test_corruption_raises_config_error(tmp_path, edit, msg):
    with pytest.raises(K.ConfigError, match=msg):
        K.read_matrix(_corrupt(tmp_path, edit))


def test_csv_plain_single_row_and_cap(tmp_path, monkeypatch):
    p = tmp_path / "m.csv"
    p.write_text("1.5,2.0\n-3.25,4.0\n")
    assert np.array_equal(K.read_csv_matrix(p), [[1.5, 2.0], [-3.25, 4.0]])
    r = tmp_path / "r.csv"
    r.write_text("1.0,2.0,3.0\n")
    assert K.read_csv_matrix(r).shape == (1, 3)
    monkeypatch.setattr(mio, "CSV_MAX_ENTRIES", 3)
    with pytest.raises(K.ConfigError):
        K.read_csv_matrix(p)
