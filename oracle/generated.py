"""Host regeneration of device-generated matrices -- ORACLE TEST
INFRASTRUCTURE ONLY (used by tests/ and bench.py's cpu_baseline leg).

`GeneratedRows(ps, q, spec)` produces row blocks bit-identical to the matrix
the device built with the same factors (include/ksvd_gen.h), so the CPU
oracle can run on configurations 3-5 (or row samples of them) through
`krylov_oracle.BlockOp`.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from oracle.build import build

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build()))
        pd = C.POINTER(C.c_double)
        _lib.ksvd_host_rows.argtypes = [pd, pd, C.c_int, C.c_int64, C.c_double, C.c_uint64,
                                        C.c_int64, C.c_int64, C.c_int, pd]
        _lib.ksvd_host_normal.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
        _lib.ksvd_host_normal.restype = C.c_double
    return _lib


def host_normal(seed: int, tag: int, idx: int) -> float:
    return float(lib().ksvd_host_normal(seed, tag, idx))


class GeneratedRows:
    def __init__(self, ps: np.ndarray, q: np.ndarray, noise: float, seed: int, f32: bool,
                 row0: int = 0):
        self.ps = np.ascontiguousarray(ps, dtype=np.float64)
        self.q = np.ascontiguousarray(q, dtype=np.float64)
        self.r = self.q.shape[1]
        self.n = self.q.shape[0]
        self.noise, self.seed, self.f32, self.row0 = float(noise), int(seed), bool(f32), row0

    def __call__(self, i0: int, i1: int) -> np.ndarray:
        """Rows [i0, i1) (global indices) as float64."""
        out = np.empty((i1 - i0, self.n))
        ps = np.ascontiguousarray(self.ps[i0 - self.row0:i1 - self.row0])
        pd = C.POINTER(C.c_double)
        lib().ksvd_host_rows(ps.ctypes.data_as(pd), self.q.ctypes.data_as(pd), self.r, self.n,
                             self.noise, self.seed, i0, i1, int(self.f32),
                             out.ctypes.data_as(pd))
        return out
