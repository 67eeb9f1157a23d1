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
        _lib.ksvd_host_gemv_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, pd, pd]
        _lib.ksvd_host_gemv_t_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, pd, pd]
        _lib.ksvd_host_gauss.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_int64, C.c_int,
                                         pd]
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


TAG_LEFT, TAG_RIGHT = 2, 3  # include/ksvd_gen.h stream tags


def host_gauss(seed: int, tag: int, row0: int, rows: int, r: int) -> np.ndarray:
    """rows x r Gaussians of the generator's factor stream, bit-identical to
    the device's k_gen_gauss (include/ksvd_gen.h)."""
    out = np.empty((rows, r))
    lib().ksvd_host_gauss(int(seed), int(tag), int(row0), int(rows), int(r),
                          out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def _cholqr2(X: np.ndarray) -> np.ndarray:
    for _ in range(2):
        L = np.linalg.cholesky(X.T @ X)
        X = np.linalg.solve(L, X.T).T
    return X


def spectrum(spec) -> np.ndarray:
    """s_1..s_r of a GenSpec (csrc/ksvd.cu generate_into)."""
    i = np.arange(1, spec.rank + 1, dtype=np.float64)
    if spec.spectrum == "harmonic":
        return spec.s0 / i
    if spec.spectrum == "exp":
        return spec.s0 * np.exp(-i / spec.p)
    if spec.rank == 1:
        return np.array([spec.s0])
    return spec.s0 * 10.0 ** (-spec.p * (i - 1) / (spec.rank - 1))


def host_generated_rows(spec, row0: int, rows: int) -> "GeneratedRows":
    """Rows [row0, row0 + rows) of a generated configuration rebuilt on the
    host alone (no GPU): the factor Gaussians are the device's bit for bit,
    the CholeskyQR2 runs in numpy, so entries agree with the device matrix
    to rounding of the orthonormal factors (~1e-15 relative), not bitwise.
    Used for the reference arm's CPU timing sample, where the values only
    have to be the configuration's."""
    r = spec.rank
    P = _cholqr2(host_gauss(spec.seed, TAG_LEFT, 0, spec.m, r))
    Q = _cholqr2(host_gauss(spec.seed, TAG_RIGHT, 0, spec.n, r))
    ps = P[row0:row0 + rows] * spectrum(spec)
    return GeneratedRows(ps, Q, spec.noise, spec.seed, spec.dtype == "f32", row0=row0)
