"""KLRM binary snapshots (reference matrixio.py:15-46).

Layout, little endian: magic ``KLRM``, u32 version 1, u64 rows, u64 cols,
then rows*cols float64 payload in row-major order.

`read_matrix_device` streams this rank's row shard of a snapshot straight
into HBM (ksvd_matrix_from_klrm: chunked reads into pinned buffers
overlapped with the host-to-device copies -- the payload never exists whole
in host memory, so snapshots larger than host RAM load fine);
`write_matrix_device` streams a device matrix back (every rank writes its
rows at their offsets).  `read_matrix` / `write_matrix` are the reference's
host functions (same names, errors and bytes).
"""

from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

from . import _lib
from .errors import ConfigError, ShapeMismatchError
from .linops import DeviceMatrix

MAGIC = b"KLRM"
VERSION = 1
HEADER_BYTES = 24  # "<4sIQQ": magic, u32 version, u64 rows, u64 cols
CSV_MAX_ENTRIES = 10 ** 6


def _header(rows: int, cols: int) -> bytes:
    return MAGIC + struct.pack("<IQQ", VERSION, rows, cols)


def _parse_header(path, head: bytes) -> tuple[int, int]:
    """Same checks and messages as the reference reader (matrixio.py:33-41)."""
    if len(head) < HEADER_BYTES:
        raise ConfigError(f"{path}: truncated header")
    if head[:4] != MAGIC:
        raise ConfigError(f"{path}: bad magic {head[:4]!r}, expected {MAGIC!r}")
    version, rows, cols = struct.unpack_from("<IQQ", head, 4)
    if version != VERSION:
        raise ConfigError(f"{path}: unsupported format version {version}")
    return rows, cols


def write_matrix(path, A) -> None:
    """Host snapshot writer (reference matrixio.py:22-29)."""
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2:
        raise ShapeMismatchError(f"can only snapshot 2-d matrices, got shape {A.shape}")
    body = np.require(A, dtype="<f8", requirements="C")
    with open(path, "wb") as f:
        f.write(_header(*A.shape))
        body.tofile(f)


def read_matrix(path) -> np.ndarray:
    """Host snapshot reader (reference matrixio.py:32-46)."""
    with open(path, "rb") as f:
        rows, cols = _parse_header(path, f.read(HEADER_BYTES))
        want = rows * cols * 8
        data = f.read(want)
    if len(data) != want:
        raise ConfigError(f"{path}: payload holds {len(data)} bytes, header promises {want}")
    out = np.empty((rows, cols), dtype=np.float64)
    out.reshape(-1)[:] = np.frombuffer(data, dtype="<f8")
    return out


def read_csv_matrix(path) -> np.ndarray:
    """Comma-separated numeric rows, capped at CSV_MAX_ENTRIES entries
    (reference matrixio.py:49-55)."""
    A = np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
    if A.size > CSV_MAX_ENTRIES:
        raise ConfigError(
            f"{path}: {A.size} entries exceeds the CSV import cap of {CSV_MAX_ENTRIES}")
    return A


def read_matrix_device(path, dtype=np.float64, ctx: _lib.Context | None = None) -> DeviceMatrix:
    """Stream a KLRM snapshot into HBM (this rank's row shard)."""
    ctx = ctx or _lib.get_context()
    dtype = np.dtype(dtype)
    if dtype not in (np.float32, np.float64):
        raise ConfigError(f"unsupported storage dtype {dtype}")
    h = C.c_void_p()
    code = _lib.KSVD_F32 if dtype == np.float32 else _lib.KSVD_F64
    _lib.check(_lib.load_library().ksvd_matrix_from_klrm(
        ctx.handle, os.fsencode(os.fspath(path)), code, C.byref(h)))
    m, n, r0, ml = (C.c_int64() for _ in range(4))
    _lib.check(_lib.load_library().ksvd_matrix_shape(h, C.byref(m), C.byref(n), C.byref(r0),
                                                     C.byref(ml), None, None))
    return DeviceMatrix(h, ctx, (m.value, n.value), r0.value, ml.value, dtype)


def write_matrix_device(path, op: DeviceMatrix) -> None:
    """Stream a device matrix to a KLRM snapshot (all ranks call it)."""
    _lib.check(_lib.load_library().ksvd_matrix_to_klrm(op.handle, os.fsencode(os.fspath(path))))
