"""Parity predicates shared by the CPU (oracle) and GPU suites.

Tolerances are the north star's (BASELINE.json): fp64 singular values to
relative error <= 1e-10 and singular vectors with sign-invariant |cos| >=
1 - 1e-8; fp32 storage to relative error <= 1e-4 and ||Av - sigma u|| <=
1e-4 sigma_1; ranks bit-exact.
"""

from __future__ import annotations

import numpy as np

SIG_RTOL_F64 = 1e-10
COS_TOL_F64 = 1e-8
SIG_RTOL_F32 = 1e-4
RES_TOL_F32 = 1e-4


def col_cos(X, Y):
    """|cos| between matching columns."""
    X = np.asarray(X)
    Y = np.asarray(Y)
    num = np.abs(np.einsum("ij,ij->j", X, Y))
    den = np.linalg.norm(X, axis=0) * np.linalg.norm(Y, axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        c = np.where(den > 0, num / den, 1.0)
    return c


def sig_relerr(s, ref):
    s = np.asarray(s)
    ref = np.asarray(ref)
    scale = np.maximum(np.abs(ref), np.finfo(float).tiny)
    return float(np.max(np.abs(s - ref) / scale)) if ref.size else 0.0


def ortho_dev(M):
    M = np.asarray(M)
    if M.shape[1] == 0:
        return 0.0
    return float(np.max(np.abs(M.T @ M - np.eye(M.shape[1]))))


def bidiagonal(alphas, betas):
    k = len(alphas)
    B = np.zeros((k + 1, k))
    i = np.arange(k)
    B[i, i] = alphas
    B[i + 1, i] = betas[1:]
    return B


def recurrence_dev(A, alphas, betas, Q, P):
    """||A P - Q B||_F / ||A||_F (reference test_bidiag.py:13-26)."""
    k = len(alphas)
    B = bidiagonal(alphas, betas)
    if Q.shape[1] == k:
        B = B[:k, :]
    dev = np.linalg.norm(np.asarray(A) @ P - Q @ B)
    return dev / max(np.linalg.norm(A), 1e-300)


def assert_scalars_close(ours_a, ours_b, ref_a, ref_b, rtol=SIG_RTOL_F64, what=""):
    assert len(ours_a) == len(ref_a), (what, len(ours_a), len(ref_a))
    assert len(ours_b) == len(ref_b), (what, len(ours_b), len(ref_b))
    if len(ref_a):
        ea = np.max(np.abs(ours_a - ref_a) / np.max(np.abs(ref_a)))
        assert ea <= rtol, (what, "alphas", ea)
    # betas: the breakdown beta is below eps and carries no relative digits
    eb = np.max(np.abs(ours_b - ref_b)) / max(np.max(np.abs(ref_b)), 1e-300)
    assert eb <= rtol, (what, "betas", eb)
