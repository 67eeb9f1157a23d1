"""Streaming KLRM ingestion into HBM row shards (ksvd_matrix_from_klrm /
ksvd_matrix_to_klrm): bit-exact against the host reader, f32 storage,
multi-chunk streaming with ragged tails, corruption errors through the
C-ABI, and a fsvd on a loaded snapshot against the oracle."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
from tests.parity import COS_TOL_F64, SIG_RTOL_F64, col_cos, sig_relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n", [(1, 1), (1, 9), (9, 1), (37, 23), (1000, 257), (4099, 33)])
def test_device_load_is_bit_exact(tmp_path, m, n):
    A = synth.gaussian_matrix(m, n, seed=m + n)
    p = tmp_path / "a.klrm"
    K.write_matrix(p, A)
    op = K.read_matrix_device(p)
    assert op.shape == (m, n) and op.dtype == np.float64
    assert np.array_equal(op.to_dense(), A)
    op32 = K.read_matrix_device(p, dtype=np.float32)
    assert op32.dtype == np.float32
    assert np.array_equal(op32.to_dense(), A.astype(np.float32))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_device_write_matches_host_writer(tmp_path, dtype):
    A = synth.gaussian_matrix(513, 70, seed=4).astype(dtype)
    ref, out = tmp_path / "ref.klrm", tmp_path / "out.klrm"
    K.write_matrix(ref, A)
    K.write_matrix_device(out, K.DeviceMatrix.from_host(A))
    assert out.read_bytes() == ref.read_bytes()
    # overwrite a larger stale file: the snapshot is truncated to size
    K.write_matrix(out, synth.gaussian_matrix(900, 90, seed=5))
    K.write_matrix_device(out, K.DeviceMatrix.from_host(A))
    assert out.read_bytes() == ref.read_bytes()


@pytest.mark.parametrize("edit,msg", [
    (lambda r: b"NOPE" + r[4:], "bad magic"),
    (lambda r: r[:4] + (7).to_bytes(4, "little") + r[8:], "unsupported format version 7"),
    (lambda r: r[:-8], "header promises"),
    (lambda r: r[:10], "truncated header"),
])
def test_device_reader_rejects_corruption(tmp_path, edit, msg):
    p = tmp_path / "x.klrm"
    K.write_matrix(p, np.eye(5))
    bad = tmp_path / "bad.klrm"
    bad.write_bytes(edit(p.read_bytes()))
    with pytest.raises(K.ConfigError, match=msg):
        K.read_matrix_device(bad)
    with pytest.raises(K.ConfigError):
        K.read_matrix_device(tmp_path / "missing.klrm")


def test_fsvd_on_loaded_snapshot(tmp_path):
    A = synth.low_rank_synth(2000, 600, 40, seed=11)
    p = tmp_path / "lr.klrm"
    K.write_matrix(p, A)
    cfg = K.BidiagConfig(k_max=60, seed=2)
    ours = K.fsvd(K.read_matrix_device(p), k=60, r=10, cfg=cfg)
    ref = O.fsvd_oracle(A, 60, 10, seed=2)
    assert sig_relerr(ours.sigma, ref.sigma) <= SIG_RTOL_F64
    assert np.min(col_cos(ours.U, ref.U)) >= 1 - COS_TOL_F64
    assert K.estimate_rank(K.read_matrix_device(p)).rank == 40


_CHUNK_SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r})
import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth
ok = []
for m, n in [(1000, 257), (777, 1025), (5, 3000)]:
    A = synth.gaussian_matrix(m, n, seed=m)
    K.write_matrix({tmp!r} + "/c.klrm", A)
    ok.append(bool(np.array_equal(K.read_matrix_device({tmp!r} + "/c.klrm").to_dense(), A)))
    ok.append(bool(np.array_equal(
        K.read_matrix_device({tmp!r} + "/c.klrm", dtype=np.float32).to_dense(),
        A.astype(np.float32))))
    K.write_matrix_device({tmp!r} + "/d.klrm", K.DeviceMatrix.from_host(A))
    ok.append(open({tmp!r} + "/d.klrm", "rb").read() == open({tmp!r} + "/c.klrm", "rb").read())
print(json.dumps(ok))
"""


def test_small_chunks_stream_ragged_tails(tmp_path):
    """4 KiB staging chunks: many double-buffered chunks per shard, rows
    larger than a chunk (one row per chunk), ragged final chunks."""
    root = str(Path(__file__).resolve().parent.parent)
    res = subprocess.run([sys.executable, "-c", _CHUNK_SCRIPT.format(root=root, tmp=str(tmp_path))],
                         env={**os.environ, "KSVD_IO_CHUNK_BYTES": "4096"},
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert all(json.loads(res.stdout.strip().splitlines()[-1]))
