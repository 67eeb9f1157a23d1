"""Golub-Kahan lower bidiagonalization on the B200 (drop-in for the
reference's bidiag.py).

Recurrences (reference bidiag.py:1-12):

    A p_i       = alpha_i q_i + beta_{i+1} q_{i+1}
    A^T q_{i+1} = beta_{i+1} p_i + alpha_{i+1} p_{i+1}

The whole loop -- both products, CGS2 against both bases, the breakdown
tests -- runs on the device inside one ksvd_gk_run call; the bases never
leave HBM unless a caller asks for them (BidiagState.Q / .P, as returned by
`bidiagonalize`).  The host contributes exactly what the reference's
contract pins bit for bit: the start vector from
substream(seed, GK_START) (bidiag.py:126-131) and, on the rare beta
breakdown, the fresh draws of the terminal column (bidiag.py:95-108).
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import math
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError
from .linops import GK_START, DeviceMatrix, as_operator, shape_of, substream


@dataclass(frozen=True)
class BidiagConfig:
    """Knobs of one run -- same fields, defaults and validation as the
    reference (bidiag.py:25-52)."""

    k_max: int
    eps: float = 1e-8
    reorth_passes: int = 2
    start_mean: float = 2.0
    start_std: float = 1.0
    seed: int = 0

    def __post_init__(self):
        if self.k_max < 1:
            raise ConfigError(f"k_max must be >= 1, got {self.k_max}")
        if not self.eps > 0:
            raise ConfigError(f"eps must be > 0, got {self.eps}")
        if self.reorth_passes not in (1, 2):
            raise ConfigError(f"reorth_passes must be 1 or 2, got {self.reorth_passes}")
        if not self.start_std > 0:
            raise ConfigError(f"start_std must be > 0, got {self.start_std}")


@dataclass(frozen=True)
class BidiagState:
    """Outcome of a run with k_prime iterations (reference bidiag.py:55-74):
    alphas (k'), betas (k'+1, betas[0] = start-vector norm), Q m x (k'+1)
    (m x k' when the left space is exhausted), P n x k'."""

    alphas: np.ndarray
    betas: np.ndarray
    Q: np.ndarray
    P: np.ndarray
    k_prime: int
    terminated_early: bool
    degenerate: bool = False


def with_k_max(cfg: BidiagConfig, k_max: int) -> BidiagConfig:
    if cfg.k_max == k_max:
        return cfg
    return dataclasses.replace(cfg, k_max=k_max)


def _free_run(handle):
    _lib.load_library().ksvd_run_free(handle)


class GKRun:
    """Device-resident result of one GK run (the bases stay in HBM)."""

    def __init__(self, handle, op: DeviceMatrix, alphas, betas, k_prime, early,
                 degenerate, q_cols):
        self.handle = handle
        self.op = op
        self.alphas = alphas
        self.betas = betas
        self.k_prime = int(k_prime)
        self.terminated_early = bool(early)
        self.degenerate = bool(degenerate)
        self.q_cols = int(q_cols)
        self._fin = weakref.finalize(self, _free_run, handle)

    def bases(self):
        """Download Q (local rows x q_cols) and P (n x k') -- the reference's
        BidiagState copies (bidiag.py:180-184)."""
        ml, n = self.op.m_local, self.op.shape[1]
        kp = self.k_prime
        Qb = np.empty((self.q_cols, ml))
        Pb = np.empty((kp, n))
        _lib.check(_lib.load_library().ksvd_run_bases(
            self.handle, _lib.dptr(Qb), self.q_cols, _lib.dptr(Pb), kp))
        return Qb.T, Pb.T

    def state(self) -> BidiagState:
        Q, P = self.bases()
        return BidiagState(alphas=self.alphas, betas=self.betas, Q=Q, P=P,
                           k_prime=self.k_prime, terminated_early=self.terminated_early,
                           degenerate=self.degenerate)

    def free(self):
        self._fin()


def _host_norm(v: np.ndarray) -> float:
    """np.linalg.norm (the reference's call) on ONE BLAS thread.  OpenBLAS
    threads its dot product above 10k elements, and its idle workers then
    spin for ~0.1 s on every core -- measured: the next staged upload of A
    (8 host copy threads) ran 2-3x slower (0.8 GB in 44-81 ms instead of
    17-20 ms).  Single-threaded it is the reference's own result on a
    one-thread BLAS (below 10k elements, the golden start vectors, it is
    bit-identical either way)."""
    lim = _blas_single() if v.size > 8192 else None  # below: never threaded
    if lim is None:
        return float(np.linalg.norm(v))
    with lim.limit(limits=1, user_api="blas"):
        return float(np.linalg.norm(v))


_CTL = []


def _blas_single():
    if not _CTL:
        try:
            from threadpoolctl import ThreadpoolController

            _CTL.append(ThreadpoolController())
        except Exception:  # noqa: BLE001 -- optional: plain numpy without it
            _CTL.append(None)
    return _CTL[0]


def _start_vector(cfg: BidiagConfig, m: int):
    # bidiag.py:126-131: q = mean + std * N(0,1) from the GK_START stream
    rng = substream(cfg.seed, GK_START)
    q = cfg.start_mean + cfg.start_std * rng.standard_normal(m)
    beta1 = _host_norm(q)
    if beta1 == 0.0:
        raise NumericalError("start vector has zero norm")
    q /= beta1
    return rng, q, beta1


def run_gk(op: DeviceMatrix, cfg: BidiagConfig) -> GKRun:
    """The GK loop of bidiag.py:111-178 on the device."""
    m, n = op.shape
    if not 1 <= cfg.k_max <= min(m, n):
        raise ConfigError(
            f"k_max must be in [1, min(m,n)] = [1, {min(m, n)}], got {cfg.k_max}")
    rng, q, beta1 = _start_vector(cfg, m)
    q_local = np.ascontiguousarray(q[op.row0:op.row0 + op.m_local])
    lib = _lib.load_library()
    h = C.c_void_p()
    _lib.check(lib.ksvd_gk_run(op.handle, int(cfg.k_max), float(cfg.eps),
                               int(cfg.reorth_passes), _lib.dptr(q_local), C.byref(h)))
    try:
        kp, flags = C.c_int(), C.c_int()
        alphas = np.empty(cfg.k_max)
        betas = np.empty(cfg.k_max + 1)
        _lib.check(lib.ksvd_run_info(h, C.byref(kp), C.byref(flags), _lib.dptr(alphas),
                                     _lib.dptr(betas)))
        kp, flags = kp.value, flags.value
        betas[0] = beta1
        degenerate = bool(flags & _lib.RUN_DEGENERATE)
        if degenerate:
            return GKRun(h, op, np.zeros(0), betas[:1].copy(), 0, True, True, 1)
        q_cols = kp + 1
        if flags & _lib.RUN_BETA_BREAK:
            if kp < m:
                _terminal_column(lib, h, op, float(betas[kp]), rng)
            else:
                q_cols = kp  # left space exhausted, Q stays square
        return GKRun(h, op, alphas[:kp].copy(), betas[:kp + 1].copy(), kp,
                     bool(flags & _lib.RUN_EARLY), False, q_cols)
    except BaseException:
        lib.ksvd_run_free(h)
        raise


def _terminal_column(lib, h, op: DeviceMatrix, beta: float, rng) -> None:
    # bidiag.py:95-108: normalised residual, else up to two fresh draws from
    # the same GK_START stream; each candidate is CGS2'd on the device and
    # kept once its norm exceeds 0.5
    m = op.shape[0]
    v_local, nrm = None, beta
    for _ in range(3):
        if nrm > 0 and math.isfinite(nrm):
            acc = C.c_int()
            _lib.check(lib.ksvd_run_extend(h, _lib.dptr(v_local), float(nrm), C.byref(acc)))
            if acc.value:
                return
        v = rng.standard_normal(m)
        nrm = _host_norm(v)
        v_local = np.ascontiguousarray(v[op.row0:op.row0 + op.m_local])
    raise NumericalError("could not extend the left basis to k'+1 columns")


def bidiagonalize(A, cfg: BidiagConfig) -> BidiagState:
    """Run the recurrence until k_max iterations or breakdown (reference
    bidiag.py:111-184); returns host copies of the bases like the reference."""
    m, n = shape_of(A)
    if not 1 <= cfg.k_max <= min(m, n):
        raise ConfigError(
            f"k_max must be in [1, min(m,n)] = [1, {min(m, n)}], got {cfg.k_max}")
    run = run_gk(as_operator(A), cfg)
    try:
        return run.state()
    finally:
        run.free()


def bidiagonal_matrix(state: BidiagState) -> np.ndarray:
    """Dense B (k'+1) x k': alphas on the diagonal, betas[1:] below it."""
    k = state.k_prime
    B = np.zeros((k + 1, k))
    idx = np.arange(k)
    B[idx, idx] = state.alphas
    B[idx + 1, idx] = state.betas[1:]
    return B
