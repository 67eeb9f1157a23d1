"""ctypes binding of libksvd.so (include/ksvd.h) and the per-process context.

There is no CPU fallback: if the library is missing or no GPU is visible,
every entry point that computes raises.  Status codes map onto the
reference's exception types (linops.py:26-35): 2 -> ConfigError,
3 -> NumericalError, anything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import ConfigError, NumericalError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libksvd.so"

KSVD_OK, KSVD_ERUNTIME, KSVD_ECONFIG, KSVD_ENUMERIC = 0, 1, 2, 3
KSVD_F64, KSVD_F32 = 0, 1
PX_HANDLE_BYTES = 64
RUN_EARLY, RUN_DEGENERATE, RUN_BETA_BREAK, RUN_ALPHA_BREAK = 1, 2, 4, 8
NCCL_UID_BYTES = 128

_vp = C.c_void_p
_i64 = C.c_int64
_pi64 = C.POINTER(C.c_int64)
_pd = C.POINTER(C.c_double)
_pi = C.POINTER(C.c_int)

class GenSpec(C.Structure):
    """ksvd_gen_spec (include/ksvd.h)."""

    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("rank", C.c_int32), ("dtype", C.c_int32),
                ("seed", C.c_uint64), ("spectrum", C.c_int32), ("pad", C.c_int32),
                ("s0", C.c_double), ("p", C.c_double), ("noise", C.c_double)]


SPEC_HARMONIC, SPEC_EXP, SPEC_GEOM = 0, 1, 2

# name -> (restype, argtypes); mirrors include/ksvd.h one to one
SIGNATURES = {
    "ksvd_last_error": (C.c_char_p, []),
    "ksvd_version": (C.c_int, []),
    "ksvd_device_count": (C.c_int, [_pi]),
    "ksvd_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "ksvd_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)]),
    "ksvd_ctx_destroy": (C.c_int, [_vp]),
    "ksvd_ctx_sync": (C.c_int, [_vp]),
    "ksvd_ctx_release_pool": (C.c_int, [_vp]),
    "ksvd_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "ksvd_ctx_kernel_stats": (C.c_int, [_vp, C.c_int, _pi64, _pd]),
    "ksvd_ctx_reset_stats": (C.c_int, [_vp]),
    "ksvd_ctx_launch_count": (C.c_int, [_vp, _pi64]),
    "ksvd_ctx_mark": (C.c_int, [_vp, C.c_int]),
    "ksvd_ctx_elapsed": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "ksvd_matrix_from_host": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i64, C.c_int,
                                        C.POINTER(_vp)]),
    "ksvd_matrix_from_device": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i64, C.c_int,
                                          C.POINTER(_vp)]),
    "ksvd_matrix_free": (C.c_int, [_vp]),
    "ksvd_matrix_shape": (C.c_int, [_vp, _pi64, _pi64, _pi64, _pi64, _pi, _pi64]),
    "ksvd_matrix_to_host": (C.c_int, [_vp, _vp]),
    "ksvd_matvec": (C.c_int, [_vp, _pd, _pd]),
    "ksvd_rmatvec": (C.c_int, [_vp, _pd, _pd]),
    "ksvd_matmat": (C.c_int, [_vp, _pd, C.c_int, _pd]),
    "ksvd_gk_run": (C.c_int, [_vp, C.c_int, C.c_double, C.c_int, _pd, C.POINTER(_vp)]),
    "ksvd_run_info": (C.c_int, [_vp, _pi, _pi, _pd, _pd]),
    "ksvd_run_extend": (C.c_int, [_vp, _pd, C.c_double, _pi]),
    "ksvd_run_bases": (C.c_int, [_vp, _pd, C.c_int, _pd, C.c_int]),
    "ksvd_ritz": (C.c_int, [_vp, _pd, _pd, C.c_int, C.c_int, _pd, _pd, _pi]),
    "ksvd_run_free": (C.c_int, [_vp]),
    "ksvd_symtridiag_eig": (C.c_int, [C.c_int, _pd, _pd, C.c_int, _pd, _pd]),
    "ksvd_bidiag_sv2": (C.c_int, [C.c_int, _pd, _pd, _pd]),
    "ksvd_matrix_generate": (C.c_int, [_vp, C.POINTER(GenSpec), C.POINTER(_vp)]),
    "ksvd_matrix_gen_factors": (C.c_int, [_vp, _pd, _pd, _pi]),
    "ksvd_matrix_from_klrm": (C.c_int, [_vp, C.c_char_p, C.c_int, C.POINTER(_vp)]),
    "ksvd_matrix_to_klrm": (C.c_int, [_vp, C.c_char_p]),
    "ksvd_dense_svd": (C.c_int, [C.c_int, _pd, _pd, _pd, _pd]),
    "ksvd_dense_svd_dev": (C.c_int, [_vp, C.c_int, _pd, _pd, _pd, _pd]),
    "ksvd_px_export": (C.c_int, [_vp, C.c_int64, C.c_char_p]),
    "ksvd_px_open": (C.c_int, [_vp, C.c_char_p]),
    "ksvd_px_enabled": (C.c_int, [_vp, _pi]),
    "ksvd_run_restart": (C.c_int, [_vp, C.c_int, _pd, _pd, C.c_int]),
    "ksvd_run_ritz_bases": (C.c_int, [_vp, _pd, C.c_int, _pd, C.c_int, C.c_int, _pd, _pd]),
    "ksvd_matrix_from_factors": (C.c_int, [_vp, _pd, _pd, _pd, C.c_int64, C.c_int64, C.c_int64,
                                           C.c_int64, C.c_int64, C.c_int64, C.POINTER(_vp)]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: Path | str | None = None) -> C.CDLL:
    """Load libksvd.so (once).  Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # KSVD_LIB_PATH: load another build of the library (A/B measurements)
        p = Path(path) if path else Path(os.environ.get("KSVD_LIB_PATH", LIB_PATH))
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build it with `python -m paper_2104_10785_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == KSVD_OK:
        return
    msg = load_library().ksvd_last_error().decode(errors="replace")
    if rc == KSVD_ECONFIG:
        raise ConfigError(msg)
    if rc == KSVD_ENUMERIC:
        raise NumericalError(msg)
    raise RuntimeError(f"libksvd: {msg}")


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_pd)


class Context:
    """One GPU (and, for nranks > 1, one NCCL communicator) per process."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1,
                 uid: bytes | None = None):
        lib = load_library()
        h = _vp()
        check(lib.ksvd_ctx_create(int(device), int(rank), int(nranks), uid, C.byref(h)))
        self.handle = h
        self.device, self.rank, self.nranks = int(device), int(rank), int(nranks)

    def close(self):
        if self.handle:
            load_library().ksvd_ctx_destroy(self.handle)
            self.handle = None

    def sync(self):
        check(load_library().ksvd_ctx_sync(self.handle))

    def release_pool(self):
        """Return freed device pool memory (e.g. after freeing a large matrix)."""
        check(load_library().ksvd_ctx_release_pool(self.handle))

    # ---- measurement hooks (bench.py) ----
    def set_profiling(self, on: bool):
        check(load_library().ksvd_ctx_set_profiling(self.handle, int(bool(on))))

    def kernel_stats(self, cls: int) -> tuple[int, float]:
        n, ms = C.c_int64(), C.c_double()
        check(load_library().ksvd_ctx_kernel_stats(self.handle, cls, C.byref(n), C.byref(ms)))
        return int(n.value), float(ms.value)

    def reset_stats(self):
        check(load_library().ksvd_ctx_reset_stats(self.handle))

    def launch_count(self) -> int:
        n = C.c_int64()
        check(load_library().ksvd_ctx_launch_count(self.handle, C.byref(n)))
        return int(n.value)

    def mark(self, slot: int):
        check(load_library().ksvd_ctx_mark(self.handle, slot))

    def elapsed_ms(self, s0: int, s1: int) -> float:
        ms = C.c_float()
        check(load_library().ksvd_ctx_elapsed(self.handle, s0, s1, C.byref(ms)))
        return float(ms.value)

    # ---- NVLink peer exchange (dist.init_distributed(peer_exchange=True)) ----
    def px_export(self, slot: int) -> bytes:
        buf = C.create_string_buffer(PX_HANDLE_BYTES)
        check(load_library().ksvd_px_export(self.handle, int(slot), buf))
        return buf.raw

    def px_open(self, handles: bytes) -> bool:
        check(load_library().ksvd_px_open(self.handle, handles))
        return self.px_enabled()

    def px_enabled(self) -> bool:
        on = C.c_int()
        check(load_library().ksvd_px_enabled(self.handle, C.byref(on)))
        return bool(on.value)


_ctx: Context | None = None


def set_context(ctx: Context | None) -> None:
    global _ctx
    _ctx = ctx


def get_context() -> Context:
    """The process context; created on first use on LOCAL_RANK's device."""
    global _ctx
    if _ctx is None:
        lib = load_library()
        n = C.c_int()
        check(lib.ksvd_device_count(C.byref(n)))
        if n.value < 1:
            raise RuntimeError("libksvd: no CUDA device visible (there is no CPU fallback)")
        dev = int(os.environ.get("LOCAL_RANK", "0")) % n.value
        _ctx = Context(device=dev)
    return _ctx


def device_count() -> int:
    """CUDA devices visible to this process (0 when none or no driver)."""
    n = C.c_int()
    try:
        check(load_library().ksvd_device_count(C.byref(n)))
    except RuntimeError:
        return 0
    return int(n.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(NCCL_UID_BYTES)
    check(load_library().ksvd_nccl_unique_id(buf))
    return buf.raw


def symtridiag_eig_native(diag: np.ndarray, off: np.ndarray, vectors: bool):
    n = int(diag.shape[0])
    d = np.ascontiguousarray(diag, dtype=np.float64)
    e = np.ascontiguousarray(off, dtype=np.float64)
    if e.shape[0] == 0:
        e = np.zeros(1)
    theta = np.empty(max(n, 1))
    G = np.empty((n, n)) if vectors and n > 0 else None
    check(load_library().ksvd_symtridiag_eig(n, dptr(d), dptr(e), int(bool(vectors)),
                                             dptr(theta), dptr(G)))
    # G holds columns contiguously (column k at G[k*n]); transpose the view
    return theta[:n], (G.T if G is not None else None)


def bidiag_sv2(alphas: np.ndarray, betas: np.ndarray) -> np.ndarray:
    """Squared singular values (descending) of the (k+1) x k lower bidiagonal
    with the given alphas (k) and betas (k+1; betas[0] unused), each to high
    relative accuracy (eig.cpp ksvd_bidiag_sv2)."""
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    k = int(a.shape[0])
    theta = np.empty(max(k, 1))
    check(load_library().ksvd_bidiag_sv2(k, dptr(a), dptr(b), dptr(theta)))
    return theta[:k]
