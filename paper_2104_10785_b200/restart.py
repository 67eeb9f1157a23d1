"""Restarted Golub-Kahan: thick restart with Ritz vectors (SURVEY.md 8(f)
row 3).  An opt-in mode BEYOND the reference's semantics -- the reference
lists restarts as a non-goal -- so its parity is against the
CPU restatement in oracle/restarted.py and against the dense SVD, not
against the reference.

Form.  After a cycle of k steps the device holds (bidiag.py's recurrence)

    A^T Q_k = P_k T,      A P_k = Q_k T^T + beta_{k+1} q_{k+1} e_k^T,

with T (k x k) upper bidiagonal (alphas on the diagonal, betas above).
With T = Uh diag(s) Vh^T the Ritz triplets are u_i = Q_k Vh e_i,
v_i = P_k Uh e_i: A^T u_i = s_i v_i exactly and
A v_i = s_i u_i + rho_i q_{k+1}, rho_i = beta_{k+1} Uh[k-1, i] -- the
residual used as the convergence test.  A restart keeps l triplets:
Q <- [u_1..u_l, q_{k+1}], P <- [v_1..v_l], and ksvd_run_restart resumes the
device loop at step l+1 (z = A^T q_{k+1}, CGS2 against the kept v's --
whose coefficients are exactly the rho_i -- then the standard steps).  The
next T is [[diag(s_l), rho], [0, alpha_{l+1}]] followed by the bidiagonal
continuation.  Each cycle costs k - l GK steps on the device (2 passes
over A each) plus a k x k dense SVD on the host (ksvd_dense_svd).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bidiag import BidiagConfig, run_gk, with_k_max
from .errors import ConfigError
from .linops import PartialSvd, as_operator, shape_of

DROP_REL = 1e-14  # same floor as fsvd (reference fsvd.py:22)


@dataclass(frozen=True)
class RestartInfo:
    restarts: int
    gk_steps: int            # device GK steps over all cycles
    residuals: np.ndarray    # ||A v_i - s_i u_i|| = |rho_i| of the returned triplets
    converged: bool
    k_prime: int             # size of the final projected matrix


def dense_svd(T: np.ndarray, ctx: _lib.Context | None = None):
    """(Uh, s, Vh) of a small square matrix: host Jacobi (ksvd_dense_svd), or
    the one-CTA device kernel when a context is given (ksvd_dense_svd_dev;
    measured slower at these sizes -- 29 latency-bound rounds per sweep --
    so fsvd_restarted uses the host routine)."""
    k = T.shape[0]
    Tc = _colmajor(T)
    Ut, Vt, s = np.empty((k, k)), np.empty((k, k)), np.empty(k)
    lib = _lib.load_library()
    if ctx is not None:
        _lib.check(lib.ksvd_dense_svd_dev(ctx.handle, k, _lib.dptr(Tc), _lib.dptr(Ut),
                                          _lib.dptr(s), _lib.dptr(Vt)))
    else:
        _lib.check(lib.ksvd_dense_svd(k, _lib.dptr(Tc), _lib.dptr(Ut), _lib.dptr(s),
                                      _lib.dptr(Vt)))
    return Ut.T, s, Vt.T


def _colmajor(X: np.ndarray) -> np.ndarray:
    """C-contiguous buffer holding X column-major (the C ABI's layout)."""
    return np.ascontiguousarray(np.asarray(X, dtype=np.float64).T)


def _info(run_handle, k_max: int):
    kp, flags = C.c_int(), C.c_int()
    a, b = np.zeros(k_max), np.zeros(k_max + 1)
    _lib.check(_lib.load_library().ksvd_run_info(run_handle, C.byref(kp), C.byref(flags),
                                                 _lib.dptr(a), _lib.dptr(b)))
    return kp.value, flags.value, a, b


def _projected(alphas, betas, kp: int, flags: int, head=None):
    """T of the current cycle and the basis column counts (kq, kp_cols).
    head = (s_l, rho) after a restart: the first l+1 columns are
    [diag(s_l), rho] over alpha_{l+1}."""
    alpha_break = bool(flags & _lib.RUN_ALPHA_BREAK)
    size = kp + 1 if alpha_break else kp
    T = np.zeros((size, size))
    l = 0
    if head is not None:
        s_l, rho = head
        l = len(s_l)
        T[:l, :l] = np.diag(s_l)
        if l < size:
            T[:l, l] = rho
    for c in range(l, min(kp, size)):
        T[c, c] = alphas[c]
        if c > l:
            T[c - 1, c] = betas[c]
    if alpha_break and kp > l:
        T[kp - 1, kp] = betas[kp]  # alpha_{k'+1} ~ 0 stays 0
    return T, size, kp


def fsvd_restarted(A, r: int, k: int | None = None, tol: float = 1e-10,
                   max_restarts: int = 100, keep: int | None = None,
                   cfg: BidiagConfig | None = None):
    """Top-r singular triplets by thick-restarted GK with a k-column basis.

    Converged when every returned triplet has ||A v - s u|| <= tol * s_1
    (A^T u - s v is zero by construction).  Returns (PartialSvd, RestartInfo).
    """
    m, n = shape_of(A)
    kmax = min(m, n)
    if not 1 <= r <= kmax:
        raise ConfigError(f"need 1 <= r <= min(m,n) = {kmax}, got r={r}")
    k = min(kmax, max(2 * r + 10, 20)) if k is None else int(k)
    if not r <= k <= kmax:
        raise ConfigError(f"need r <= k <= min(m,n); got r={r}, k={k}, min(m,n)={kmax}")
    l_keep = min(k - 1, max(r, (k + r) // 2)) if keep is None else int(keep)
    if k < kmax and not r <= l_keep < k:
        raise ConfigError(f"keep must be in [r, k); got keep={l_keep}, r={r}, k={k}")
    if not tol > 0:
        raise ConfigError(f"tol must be > 0, got {tol}")
    cfg = BidiagConfig(k_max=k) if cfg is None else with_k_max(cfg, k)
    op = as_operator(A)
    run = run_gk(op, cfg)
    lib = _lib.load_library()
    try:
        if run.degenerate:
            empty = PartialSvd(np.zeros((op.m_local, 0)), np.zeros(0), np.zeros((n, 0)),
                               truncated=True, n_dropped=0)
            return empty, RestartInfo(0, 0, np.zeros(0), True, 0)
        kp, flags, a, b = _info(run.handle, k)
        b[0] = run.betas[0]
        head, restarts, steps = None, 0, kp
        while True:
            T, kq, kpc = _projected(a, b, kp, flags, head)
            Uh, s, Vh = dense_svd(T)  # host Jacobi: faster than the 1-CTA kernel at k <= 100
            early = bool(flags & _lib.RUN_EARLY)
            if flags & _lib.RUN_ALPHA_BREAK:
                # A v_i = s_i u_i exactly; the residual sits on the other
                # side: A^T u_i - s_i v_i = alpha_{k'+1} Vh[k', i] p_{k'+1}
                resid = abs(a[kp]) * np.abs(Vh[kp, :])
            else:
                # rho_i = beta_{k'+1} Uh[k'-1, i] (beta_{k'+1} < eps on a beta
                # breakdown: small, not zero)
                resid = abs(b[kp]) * np.abs(Uh[kp - 1, :])
            s1 = float(s[0]) if s.size else 0.0
            n_keep = int((s > DROP_REL * s1).sum())
            take = min(r, n_keep)
            converged = bool(np.all(resid[:take] <= tol * s1))
            # a breakdown exhausted the Krylov space: nothing to restart from
            if converged or early or restarts >= max_restarts or k >= kmax:
                break
            l = l_keep
            X = _colmajor(Vh[:, :l])
            Y = _colmajor(Uh[:, :l])
            head = (s[:l].copy(), b[kp] * Uh[kp - 1, :l])
            _lib.check(lib.ksvd_run_restart(run.handle, l, _lib.dptr(X), _lib.dptr(Y), k))
            restarts += 1
            kp, flags, a, b = _info(run.handle, k)
            steps += kp - l
        X = _colmajor(Vh[:kq, :take])
        Y = _colmajor(Uh[:kpc, :take])
        Ub = np.empty((take, op.m_local))
        Vb = np.empty((take, n))
        if take:
            _lib.check(lib.ksvd_run_ritz_bases(run.handle, _lib.dptr(X), kq, _lib.dptr(Y), kpc,
                                               take, _lib.dptr(Ub), _lib.dptr(Vb)))
        psvd = PartialSvd(U=Ub.T, sigma=s[:take].copy(), V=Vb.T, truncated=take < r,
                          n_dropped=r - take)
        return psvd, RestartInfo(restarts, steps, resid[:take].copy(), converged, T.shape[0])
    finally:
        run.free()
