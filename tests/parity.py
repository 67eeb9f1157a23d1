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


def gram_eigs(alphas, betas):
    """Ritz values theta of B^T B (dense eigvalsh; test-side helper)."""
    k = len(alphas)
    if k == 0:
        return np.zeros(0)
    B = bidiagonal(alphas, betas)
    return np.sort(np.linalg.eigvalsh(B.T @ B))[::-1]


def assert_gk_match(a, b, kp, ra, rb, rkp, head=8, kp_slack=2, what=""):
    """Parity of two GK runs on the same input with different summation
    orders.  The per-step scalars are forward-unstable once the Krylov space
    nears the numerical rank (the recurrence amplifies rounding; measured
    here and in SURVEY.md 8(c) probe 5), so the contract is: k' within a
    small window, the leading `head` alphas/betas to 1e-10, and the Ritz
    values of B^T B -- the quantities fsvd/estimate_rank consume -- to
    1e-10 of theta_1."""
    assert abs(kp - rkp) <= kp_slack, (what, kp, rkp)
    h = min(head, len(a), len(ra))
    if h:
        scale = np.max(np.abs(ra))
        assert np.max(np.abs(a[:h] - ra[:h])) <= SIG_RTOL_F64 * scale, (what, "alphas")
        bscale = np.max(np.abs(rb))
        assert np.max(np.abs(b[:h + 1] - rb[:h + 1])) <= SIG_RTOL_F64 * bscale, (what, "betas")
    th, rth = gram_eigs(a, b), gram_eigs(ra, rb)
    nt = min(len(th), len(rth))
    if nt:
        assert np.max(np.abs(th[:nt] - rth[:nt])) <= SIG_RTOL_F64 * rth[0], (what, "theta")


def assert_scalars_close(ours_a, ours_b, ref_a, ref_b, rtol=SIG_RTOL_F64, what=""):
    assert len(ours_a) == len(ref_a), (what, len(ours_a), len(ref_a))
    assert len(ours_b) == len(ref_b), (what, len(ours_b), len(ref_b))
    if len(ref_a):
        ea = np.max(np.abs(ours_a - ref_a) / np.max(np.abs(ref_a)))
        assert ea <= rtol, (what, "alphas", ea)
    # betas: the breakdown beta is below eps and carries no relative digits
    eb = np.max(np.abs(ours_b - ref_b)) / max(np.max(np.abs(ref_b)), 1e-300)
    assert eb <= rtol, (what, "betas", eb)
