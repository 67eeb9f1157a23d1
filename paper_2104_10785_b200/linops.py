"""Operators, streams and result types of the GK path.

`DeviceMatrix` is the plug-in: it implements the reference's
`LinearOperator` protocol (linops.py:132-150 -- shape, matvec, rmatvec,
matmat, rmatmat, to_dense) over a matrix resident in B200 HBM, so the
entry points in bidiag.py / fsvd.py / rank.py accept it where the
reference accepts any operator.  ndarrays are uploaded on the way in
(the reference coerces them to float64, linops.py:82-86; float32 input is
kept as float32 storage -- its entries are exact in float64 and every
product accumulates in float64).

Generic Python operators (e.g. a FactoredOperator) are NOT accelerated and
are rejected: there is no CPU fallback on this path.

Multi-GPU: with a distributed context (dist.py) the matrix is row-sharded
with `row_partition`; matvec / U results then hold this rank's rows.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError, ShapeMismatchError  # noqa: F401

# Stream tag of the GK start vector (reference linops.py:46).
GK_START = 4
BENCH_MATRIX, BENCH_METHOD = 12, 13  # reference linops.py:54-55 stream tags


def substream(seed: int, *path: int) -> np.random.Generator:
    """numpy Philox generator keyed by (seed, path) -- the reference's stream
    contract (linops.py:59-69), kept bit for bit so q_1 is identical."""
    if seed is None:
        raise ConfigError("seed must be a non-negative int, got None")
    seq = np.random.SeedSequence(entropy=int(seed), spawn_key=tuple(int(p) for p in path))
    return np.random.Generator(np.random.Philox(seq))


def derive_seed(seed: int, *path: int) -> int:
    """Child seed for a component that takes its own seed (reference
    linops.py:72-76): first u64 word of SeedSequence(seed, spawn_key=path)."""
    seq = np.random.SeedSequence(entropy=int(seed), spawn_key=tuple(int(p) for p in path))
    return int(seq.generate_state(1, dtype=np.uint64)[0])


def row_partition(m: int, nranks: int, rank: int) -> tuple[int, int]:
    """(row0, m_local): contiguous, balanced row shards; the first m % nranks
    ranks get one extra row."""
    base, extra = divmod(int(m), int(nranks))
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


class LinearOperator:
    """Anything with shape, matvec(x) and rmatvec(y) (reference protocol)."""

    shape: tuple[int, int]

    def matvec(self, x):
        raise NotImplementedError

    def rmatvec(self, y):
        raise NotImplementedError

    def matmat(self, X):
        return np.column_stack([self.matvec(X[:, j]) for j in range(X.shape[1])])

    def rmatmat(self, Y):
        return np.column_stack([self.rmatvec(Y[:, j]) for j in range(Y.shape[1])])

    def to_dense(self):
        raise NotImplementedError


def _free_matrix(handle):
    lib = _lib.load_library()
    lib.ksvd_matrix_free(handle)


class DeviceMatrix(LinearOperator):
    """Dense m x n matrix (this rank's row shard) in HBM, row-major, leading
    dimension padded to 16 bytes (one TMA / vector-load granule)."""

    def __init__(self, handle, ctx: _lib.Context, shape, row0: int, m_local: int,
                 dtype: np.dtype):
        self.handle = handle
        self.ctx = ctx
        self.shape = (int(shape[0]), int(shape[1]))
        self.row0, self.m_local = int(row0), int(m_local)
        self.dtype = np.dtype(dtype)
        self._fin = weakref.finalize(self, _free_matrix, handle)

    # ---- construction ----
    @classmethod
    def from_host(cls, A, ctx: _lib.Context | None = None, dtype=None,
                  rows_are_local: bool = False, m_global: int | None = None,
                  row0: int | None = None) -> "DeviceMatrix":
        """Upload A.  By default A is the full matrix and this rank takes its
        row shard; with rows_are_local=True A holds only the local rows
        [row0, row0 + A.shape[0]) of an m_global-row matrix."""
        ctx = ctx or _lib.get_context()
        A = np.asarray(A)
        if A.ndim != 2:
            raise ShapeMismatchError(f"expected a 2-d matrix, got shape {A.shape}")
        if dtype is None:
            dtype = np.float32 if A.dtype == np.float32 else np.float64
        dtype = np.dtype(dtype)
        if dtype not in (np.float32, np.float64):
            raise ConfigError(f"unsupported storage dtype {dtype}")
        if rows_are_local:
            if m_global is None or row0 is None:
                raise ConfigError("rows_are_local needs m_global and row0")
            m, n = int(m_global), int(A.shape[1])
            r0, ml = int(row0), int(A.shape[0])
            local = A
        else:
            m, n = (int(s) for s in A.shape)
            r0, ml = row_partition(m, ctx.nranks, ctx.rank)
            local = A[r0:r0 + ml]
        if local.dtype != dtype or local.strides[1] != dtype.itemsize or ml == 0:
            local = np.ascontiguousarray(local, dtype=dtype)
        src_ld = local.strides[0] // dtype.itemsize if ml > 1 else n
        if local.strides[0] % dtype.itemsize or src_ld < n:
            local = np.ascontiguousarray(local)
            src_ld = n
        h = C.c_void_p()
        code = _lib.KSVD_F32 if dtype == np.float32 else _lib.KSVD_F64
        ptr = local.ctypes.data if ml > 0 else None
        _lib.check(_lib.load_library().ksvd_matrix_from_host(
            ctx.handle, ptr, m, n, r0, ml, src_ld, code, C.byref(h)))
        return cls(h, ctx, (m, n), r0, ml, dtype)

    @classmethod
    def from_device_ptr(cls, ptr: int, m: int, n: int, src_ld: int, dtype,
                        ctx: _lib.Context | None = None, row0: int = 0,
                        m_local: int | None = None) -> "DeviceMatrix":
        """Copy local rows from device memory (e.g. a CUDA torch tensor)."""
        ctx = ctx or _lib.get_context()
        dtype = np.dtype(dtype)
        ml = m if m_local is None else int(m_local)
        h = C.c_void_p()
        code = _lib.KSVD_F32 if dtype == np.float32 else _lib.KSVD_F64
        _lib.check(_lib.load_library().ksvd_matrix_from_device(
            ctx.handle, C.c_void_p(ptr), m, n, row0, ml, src_ld, code, C.byref(h)))
        return cls(h, ctx, (m, n), row0, ml, dtype)

    @classmethod
    def from_torch(cls, t, ctx: _lib.Context | None = None, row0: int = 0,
                   m_global: int | None = None) -> "DeviceMatrix":
        """Copy a CUDA torch tensor holding this rank's rows."""
        import torch

        if not t.is_cuda or t.dim() != 2 or t.stride(1) != 1:
            raise ConfigError("expected a row-major 2-d CUDA tensor")
        dt = {torch.float64: np.float64, torch.float32: np.float32}.get(t.dtype)
        if dt is None:
            raise ConfigError(f"unsupported tensor dtype {t.dtype}")
        torch.cuda.synchronize(t.device)
        m = int(t.shape[0]) if m_global is None else int(m_global)
        return cls.from_device_ptr(t.data_ptr(), m, int(t.shape[1]), int(t.stride(0)), dt,
                                   ctx=ctx, row0=row0, m_local=int(t.shape[0]))

    # ---- protocol ----
    def _vec(self, x, n, what):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim != 1 or x.shape[0] != n:
            raise ShapeMismatchError(f"{what}: A has shape {self.shape}, got {x.shape}")
        return x

    def matvec(self, x):
        """y = A x (this rank's rows when sharded)."""
        x = self._vec(x, self.shape[1], "matvec")
        y = np.empty(self.m_local)
        _lib.check(_lib.load_library().ksvd_matvec(self.handle, _lib.dptr(x), _lib.dptr(y)))
        return y

    def rmatvec(self, y):
        """z = A^T y (y: this rank's rows when sharded; z all-reduced)."""
        y = self._vec(y, self.m_local, "rmatvec")
        z = np.empty(self.shape[1])
        _lib.check(_lib.load_library().ksvd_rmatvec(self.handle, _lib.dptr(y), _lib.dptr(z)))
        return z

    def matmat(self, X):
        X = np.asarray(X, dtype=np.float64)
        if X.ndim != 2 or X.shape[0] != self.shape[1]:
            raise ShapeMismatchError(f"matmat: A has shape {self.shape}, X has {X.shape}")
        k = X.shape[1]
        Xc = np.ascontiguousarray(X.T)  # k contiguous columns
        Y = np.empty((k, self.m_local))
        _lib.check(_lib.load_library().ksvd_matmat(self.handle, _lib.dptr(Xc), k, _lib.dptr(Y)))
        return Y.T

    def to_dense(self):
        out = np.empty((self.m_local, self.shape[1]), dtype=self.dtype)
        _lib.check(_lib.load_library().ksvd_matrix_to_host(
            self.handle, out.ctypes.data if self.m_local else None))
        return out

    def gen_factors(self):
        """(Ps_local, Q) of a device-generated matrix: Ps = P diag(s) for this
        rank's rows (m_local x r) and Q (n x r), for oracle regeneration."""
        lib = _lib.load_library()
        r = C.c_int()
        _lib.check(lib.ksvd_matrix_gen_factors(self.handle, None, None, C.byref(r)))
        ps = np.empty((self.m_local, r.value))
        q = np.empty((self.shape[1], r.value))
        _lib.check(lib.ksvd_matrix_gen_factors(self.handle, _lib.dptr(ps), _lib.dptr(q),
                                               C.byref(r)))
        return ps, q

    def free(self):
        self._fin()


class FactoredOperator(DeviceMatrix):
    """left @ core @ right^T applied without forming the product (reference
    linops.py:176-205), resident on the device.

    left is d1 x s1, core s1 x s2, right d2 x s2; products cost
    O((d1 + d2) s) per vector (ksvd_matrix_from_factors: the dense gemv
    kernels on the factors plus an s1 x s2 core product), so fsvd /
    estimate_rank / bidiagonalize run on it exactly as on a DeviceMatrix --
    the retraction caller's (manifold.py:121-130, 180) large targets never
    materialize d1 x d2.  Under a multi-rank context this rank holds its row
    shard of `left`; core and right are replicated."""

    def __init__(self, left, core, right, ctx: _lib.Context | None = None):
        left, core, right = (self._check(x) for x in (left, core, right))
        if left.shape[1] != core.shape[0] or right.shape[1] != core.shape[1]:
            raise ShapeMismatchError(
                f"factored operator: left {left.shape}, core {core.shape}, "
                f"right {right.shape} do not chain")
        ctx = ctx or _lib.get_context()
        m, n = left.shape[0], right.shape[0]
        r0, ml = row_partition(m, ctx.nranks, ctx.rank)
        rows = np.ascontiguousarray(left[r0:r0 + ml])
        core_c, right_c = np.ascontiguousarray(core), np.ascontiguousarray(right)
        h = C.c_void_p()
        _lib.check(_lib.load_library().ksvd_matrix_from_factors(
            ctx.handle, _lib.dptr(rows) if ml else None, _lib.dptr(core_c), _lib.dptr(right_c),
            m, n, core.shape[0], core.shape[1], r0, ml, C.byref(h)))
        super().__init__(h, ctx, (m, n), r0, ml, np.float64)
        self.left, self.core, self.right = left, core, right

    @staticmethod
    def _check(X) -> np.ndarray:
        X = np.asarray(X, dtype=np.float64)
        if X.ndim != 2:
            raise ShapeMismatchError(f"expected a 2-d matrix, got shape {X.shape}")
        return X

    def to_dense(self):
        """This rank's rows of left @ core @ right^T, formed on the device
        (one factored product per column)."""
        return self.matmat(np.eye(self.shape[1]))


def shape_of(A) -> tuple[int, int]:
    """(m, n) without touching the device (validation before upload)."""
    if isinstance(A, DeviceMatrix):
        return A.shape
    shp = getattr(A, "shape", None)
    if shp is None:
        shp = np.shape(A)
    if len(shp) != 2:
        raise ShapeMismatchError(f"expected a 2-d matrix, got shape {tuple(shp)}")
    return int(shp[0]), int(shp[1])


def as_operator(A) -> DeviceMatrix:
    """DeviceMatrix pass-through; ndarrays (and array-likes) are uploaded.
    Python-level operators cannot run on this path and are rejected."""
    if isinstance(A, DeviceMatrix):
        return A
    if all(hasattr(A, f) for f in ("left", "core", "right")) and hasattr(A, "matvec"):
        # the reference's FactoredOperator (linops.py:176-205): same factors
        # on the device, never formed
        return FactoredOperator(A.left, A.core, A.right)
    if isinstance(A, LinearOperator) or (hasattr(A, "matvec") and hasattr(A, "rmatvec")
                                         and not isinstance(A, np.ndarray)):
        raise ConfigError(
            f"{type(A).__name__} is a host-side operator; the B200 path needs a dense "
            "matrix (ndarray, CUDA tensor or DeviceMatrix) -- there is no CPU fallback")
    try:
        import torch

        if isinstance(A, torch.Tensor) and A.is_cuda:
            # device-to-device copy of this rank's row shard (any layout,
            # any real dtype: made row-major f64 / f32 on the device first)
            if A.dim() != 2:
                raise ShapeMismatchError(f"expected a 2-d matrix, got shape {tuple(A.shape)}")
            ctx = _lib.get_context()
            m = int(A.shape[0])
            r0, ml = row_partition(m, ctx.nranks, ctx.rank)
            # this rank's rows first: a large A on one GPU is never copied
            # whole to every rank's device, nor up-cast whole
            t = A[r0:r0 + ml]
            if t.device.index != ctx.device:
                t = t.to(f"cuda:{ctx.device}")
            if t.dtype not in (torch.float64, torch.float32):
                t = t.to(torch.float64)
            if t.dim() != 2 or (ml > 0 and t.stride(1) != 1) or (ml > 1 and t.stride(0) < t.shape[1]):
                t = t.contiguous()
            return DeviceMatrix.from_torch(t, ctx=ctx, row0=r0, m_global=m)
    except ImportError:
        pass
    A = np.asarray(A)
    if A.ndim != 2:
        raise ShapeMismatchError(f"expected a 2-d matrix, got shape {A.shape}")
    if A.dtype not in (np.float32, np.float64):
        # up-cast only this rank's rows (the reference coerces to f64, linops.py:82-86)
        ctx = _lib.get_context()
        r0, ml = row_partition(int(A.shape[0]), ctx.nranks, ctx.rank)
        return DeviceMatrix.from_host(np.asarray(A[r0:r0 + ml], dtype=np.float64), ctx=ctx,
                                      rows_are_local=True, m_global=int(A.shape[0]), row0=r0)
    return DeviceMatrix.from_host(A)


@dataclass(frozen=True)
class PartialSvd:
    """r singular triplets: A v_i ~= sigma_i u_i with sigma descending
    (reference linops.py:246-268).  Under a multi-rank context U holds this
    rank's rows."""

    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    truncated: bool = False
    n_dropped: int = 0

    @property
    def rank(self) -> int:
        return int(self.sigma.shape[0])

    def top(self, r: int) -> "PartialSvd":
        r = min(r, self.rank)
        return PartialSvd(self.U[:, :r].copy(), self.sigma[:r].copy(), self.V[:, :r].copy())
