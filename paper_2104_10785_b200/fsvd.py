"""Partial SVD from the device bidiagonalization (drop-in for the
reference's fsvd.py).

Pipeline (reference fsvd.py:158-204): GK run on the device -> Gram
tridiagonal B^T B in closed form -> eigenpairs on the host (native QL,
k' is a few hundred at most) -> Ritz selection -> ksvd_ritz on the device:
V = P G, U = A V / sigma in ONE pass over A (the reference makes `take`
separate passes), CGS2 column filter with the 1e-2 cut, sign fix.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bidiag import BidiagConfig, BidiagState, run_gk, with_k_max
from .errors import ConfigError, NumericalError
from .linops import PartialSvd, as_operator, shape_of

# Ritz values below (DROP_REL * sigma_1)^2 carry no usable direction
# (reference fsvd.py:20-22).
DROP_REL = 1e-14
# Residual cut of the left-vector filter (reference fsvd.py:137-142).
DEPENDENT_TOL = 1e-2
# k' of the most recent fsvd run in this process (bench instrumentation)
last_k_prime = 0


@dataclass(frozen=True)
class SymTridiag:
    """Symmetric tridiagonal matrix: main diagonal plus one off-diagonal."""

    diag: np.ndarray
    offdiag: np.ndarray

    def __post_init__(self):
        if self.diag.ndim != 1 or self.offdiag.ndim != 1:
            raise ConfigError("SymTridiag wants 1-d diag and offdiag")
        if self.offdiag.shape[0] != max(self.diag.shape[0] - 1, 0):
            raise ConfigError(
                f"offdiag length {self.offdiag.shape[0]} does not fit "
                f"diag length {self.diag.shape[0]}")

    def to_dense(self) -> np.ndarray:
        n = self.diag.shape[0]
        T = np.diag(self.diag)
        if n > 1:
            i = np.arange(n - 1)
            T[i, i + 1] = self.offdiag
            T[i + 1, i] = self.offdiag
        return T


def _gram(alphas: np.ndarray, betas: np.ndarray) -> SymTridiag:
    # diag_i = alpha_i^2 + beta_{i+1}^2, off_i = alpha_{i+1} beta_{i+1}
    # (reference fsvd.py:50-60)
    a, b = alphas, betas
    return SymTridiag(diag=a * a + b[1:] * b[1:], offdiag=a[1:] * b[1:-1])


def gram_tridiag(state) -> SymTridiag:
    """T = B^T B in closed form from the alpha/beta scalars."""
    if state.k_prime == 0:
        raise NumericalError("degenerate bidiagonalization (k' = 0) has no Gram matrix")
    return _gram(np.asarray(state.alphas, np.float64), np.asarray(state.betas, np.float64))


def symtridiag_eig(tri: SymTridiag, vectors: bool = True):
    """All eigenvalues (descending) and optionally eigenvectors of a
    symmetric tridiagonal matrix; native implicit-shift QL (eig.cpp) with
    the reference's deflation rule and sweep budget (fsvd.py:63-134)."""
    if tri.diag.shape[0] == 0:
        raise ConfigError("empty tridiagonal")
    return _lib.symtridiag_eig_native(tri.diag, tri.offdiag, vectors)


def fsvd(A, k: int, r: int, cfg: BidiagConfig | None = None,
         orthonormalize_u: bool = True, return_details: bool = False):
    """Top-r singular triplets from at most k GK iterations (reference
    fsvd.py:158-204; same arguments, results and flags)."""
    m, n = shape_of(A)
    if not 1 <= r <= k <= min(m, n):
        raise ConfigError(
            f"need 1 <= r <= k <= min(m,n); got r={r}, k={k}, min(m,n)={min(m, n)}")
    cfg = BidiagConfig(k_max=k) if cfg is None else with_k_max(cfg, k)
    op = as_operator(A)
    global last_k_prime
    run = run_gk(op, cfg)
    last_k_prime = run.k_prime
    try:
        if run.degenerate:
            empty = PartialSvd(np.zeros((op.m_local, 0)), np.zeros(0), np.zeros((n, 0)),
                               truncated=True, n_dropped=0)
            return (empty, run.state(), np.zeros(0)) if return_details else empty

        theta, G = symtridiag_eig(_gram(run.alphas, run.betas))
        sigma1 = math.sqrt(max(float(theta[0]), 0.0))
        floor = (DROP_REL * sigma1) ** 2
        n_keep = int((theta > floor).sum())  # descending: a prefix
        take = min(r, n_keep)
        sig = np.sqrt(theta[:take])

        kp = run.k_prime
        Gt = np.ascontiguousarray(G[:, :take].T)  # take contiguous columns of k'
        Ub = np.empty((take, op.m_local))
        Vb = np.empty((take, n))
        good = C.c_int()
        _lib.check(_lib.load_library().ksvd_ritz(
            run.handle, _lib.dptr(Gt), _lib.dptr(np.ascontiguousarray(sig)), take,
            int(bool(orthonormalize_u)), _lib.dptr(Ub), _lib.dptr(Vb), C.byref(good)))
        if good.value < take:
            take = good.value
            sig = sig[:take]
        U, V = Ub[:take].T, Vb[:take].T
        psvd = PartialSvd(U=U, sigma=sig, V=V, truncated=take < r,
                          n_dropped=min(r, kp) - take)
        if return_details:
            return psvd, run.state(), theta
        return psvd
    finally:
        run.free()
