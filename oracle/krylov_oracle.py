"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm for the GK hot path
(krysvd, arXiv 2104.10785), used as the checker by tests/, by
__graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
leg.  Nothing in paper_2104_10785_b200/ imports it; the product path has no
CPU fallback.

Every function cites the reference lines it restates.  Arithmetic runs in
float64 through numpy/OpenBLAS exactly where the reference does (products,
CGS2 matmuls, norms), so its results match the reference up to BLAS
summation order.  Pinning: tests/test_oracle_golden.py checks this module
against golden vectors produced by the reference itself
(tests/golden/make_golden.py, run in the build container where
/root/reference is importable) and against the reference's own known-answer
tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GK_START = 4  # reference linops.py:46
DROP_REL = 1e-14  # reference fsvd.py:22
DEPENDENT_TOL = 1e-2  # reference fsvd.py:142


class OracleConfigError(ValueError):
    pass


class OracleNumericalError(RuntimeError):
    pass


def philox_stream(seed: int, tag: int) -> np.random.Generator:
    """numpy Philox keyed by SeedSequence(seed, spawn_key=(tag,))
    (reference linops.py:59-69)."""
    return np.random.Generator(
        np.random.Philox(np.random.SeedSequence(entropy=int(seed), spawn_key=(int(tag),))))


class DenseOp:
    """Row-major float64 matrix behind apply / apply_t (linops.py:160-164)."""

    def __init__(self, A):
        self.A = np.asarray(A, dtype=np.float64)  # linops.py:82-86 coercion
        self.shape = self.A.shape

    def apply(self, x):
        return self.A @ x

    def apply_t(self, y):
        return self.A.T @ y

    def apply_many(self, X):
        return self.A @ X


class BlockOp:
    """Matrix-free operator over row blocks produced on demand (rows(i0,i1)
    -> float64 block); for oracles of generated matrices too large to hold."""

    def __init__(self, m, n, rows, block=4096):
        self.shape = (int(m), int(n))
        self.rows = rows
        self.block = int(block)

    def apply(self, x):
        m = self.shape[0]
        y = np.empty(m)
        for i0 in range(0, m, self.block):
            i1 = min(m, i0 + self.block)
            y[i0:i1] = self.rows(i0, i1) @ x
        return y

    def apply_t(self, y):
        z = np.zeros(self.shape[1])
        for i0 in range(0, self.shape[0], self.block):
            i1 = min(self.shape[0], i0 + self.block)
            z += self.rows(i0, i1).T @ y[i0:i1]
        return z

    def apply_many(self, X):
        return np.column_stack([self.apply(X[:, j]) for j in range(X.shape[1])])


def as_op(A):
    return A if hasattr(A, "apply") else DenseOp(A)


@dataclass
class GKResult:
    alphas: np.ndarray
    betas: np.ndarray
    Q: np.ndarray
    P: np.ndarray
    k_prime: int
    terminated_early: bool
    degenerate: bool = False
    breakdown: str = ""  # "", "beta", "alpha"
    steps_done: int = 0  # products of each kind performed
    timings: dict = field(default_factory=dict)


def _reorth(v, basis, passes):
    # classical Gram-Schmidt applied `passes` times (bidiag.py:77-87)
    for _ in range(passes):
        if basis.shape[1]:
            v = v - basis @ (basis.T @ v)
    return v


def _finite_or_raise(v, label):
    # bidiag.py:90-92
    if not np.isfinite(v).all():
        raise OracleNumericalError(f"non-finite values encountered in {label}")


def gk_oracle(A, k_max, eps=1e-8, reorth_passes=2, start_mean=2.0, start_std=1.0,
              seed=0) -> GKResult:
    """Golub-Kahan lower bidiagonalisation with CGS2, breakdown handling and
    terminal-column completion (bidiag.py:111-184, 95-108)."""
    op = as_op(A)
    m, n = op.shape
    if not 1 <= k_max <= min(m, n):
        raise OracleConfigError(f"k_max must be in [1, {min(m, n)}], got {k_max}")
    rng = philox_stream(seed, GK_START)
    # start vector (bidiag.py:126-131)
    q = start_mean + start_std * rng.standard_normal(m)
    nq = float(np.linalg.norm(q))
    if nq == 0.0:
        raise OracleNumericalError("start vector has zero norm")
    q /= nq
    left = np.empty((m, k_max + 1))
    right = np.empty((n, k_max))
    left[:, 0] = q
    a_list, b_list = [], [nq]

    # first right vector (bidiag.py:139-147)
    z = op.apply_t(q)
    _finite_or_raise(z, "A^T q_1")
    a = float(np.linalg.norm(z))
    if a < eps:
        return GKResult(np.zeros(0), np.array(b_list), left[:, :1].copy(),
                        right[:, :0].copy(), 0, True, degenerate=True, steps_done=0)
    right[:, 0] = z / a
    a_list.append(a)

    kp, early, why = k_max, False, ""
    for i in range(1, k_max + 1):
        # left half-step (bidiag.py:152-165)
        w = op.apply(right[:, i - 1]) - a_list[-1] * left[:, i - 1]
        _finite_or_raise(w, f"A p_{i}")
        w = _reorth(w, left[:, :i], reorth_passes)
        b = float(np.linalg.norm(w))
        b_list.append(b)
        if b < eps:
            kp, early, why = i, True, "beta"
            if i < m:
                left[:, i] = _complete_left(w, b, left[:, :i], rng)
            else:
                left = left[:, :i]
            break
        left[:, i] = w / b
        if i == k_max:  # stop before alpha_{k+1} (bidiag.py:166-168)
            break
        # right half-step (bidiag.py:169-178)
        z = op.apply_t(left[:, i]) - b * right[:, i - 1]
        _finite_or_raise(z, f"A^T q_{i + 1}")
        z = _reorth(z, right[:, :i], reorth_passes)
        a = float(np.linalg.norm(z))
        if a < eps:
            kp, early, why = i, True, "alpha"
            break
        right[:, i] = z / a
        a_list.append(a)
    ncols = min(kp + 1, left.shape[1])
    return GKResult(np.array(a_list, dtype=np.float64), np.array(b_list, dtype=np.float64),
                    left[:, :ncols].copy(), right[:, :kp].copy(), kp, early,
                    breakdown=why, steps_done=kp)


def _complete_left(w, beta, basis, rng):
    # bidiag.py:95-108: normalised residual first, then fresh draws from the
    # same stream; accept once the re-orthogonalised norm exceeds 0.5
    cand, scale = w, beta
    for _ in range(3):
        if scale > 0 and np.isfinite(scale):
            v = _reorth(cand / scale, basis, 2)
            nv = float(np.linalg.norm(v))
            if nv > 0.5:
                return v / nv
        cand = rng.standard_normal(w.shape[0])
        scale = float(np.linalg.norm(cand))
    raise OracleNumericalError("could not extend the left basis to k'+1 columns")


def gram_of(alphas, betas):
    """Closed-form B^T B (fsvd.py:50-60): (diag, offdiag)."""
    a = np.asarray(alphas, np.float64)
    b = np.asarray(betas, np.float64)
    return a * a + b[1:] ** 2, a[1:] * b[1:-1]


def ql_eig(diag, off, vectors=True):
    """Implicit-shift QL on a symmetric tridiagonal (fsvd.py:63-134):
    deflate where |e_m| <= eps (|d_m| + |d_{m+1}|), 64 sweeps per
    eigenvalue, stable descending order."""
    n = len(diag)
    if n == 0:
        raise OracleConfigError("empty tridiagonal")
    d = [float(x) for x in diag]
    e = [float(x) for x in off] + [0.0]
    Z = np.eye(n) if vectors else None
    ulp = float(np.finfo(np.float64).eps)
    for l in range(n):
        sweeps = 0
        while True:
            if sweeps == 64:  # the reference checks at most 64 times
                raise OracleNumericalError("tridiagonal QL did not converge in 64 sweeps")
            m = l
            while m < n - 1 and abs(e[m]) > ulp * (abs(d[m]) + abs(d[m + 1])):
                m += 1
            if m == l:
                break
            sweeps += 1
            g = (d[l + 1] - d[l]) / (2.0 * e[l])
            rr = math.hypot(g, 1.0)
            g = d[m] - d[l] + e[l] / (g + math.copysign(rr, g))
            s = c = 1.0
            p = 0.0
            hit_zero = False
            i = m - 1
            while i >= l:
                f, bb = s * e[i], c * e[i]
                rr = math.hypot(f, g)
                e[i + 1] = rr
                if rr == 0.0:
                    d[i + 1] -= p
                    e[m] = 0.0
                    hit_zero = True
                    break
                s, c = f / rr, g / rr
                g = d[i + 1] - p
                rr = (d[i] - g) * s + 2.0 * c * bb
                p = s * rr
                d[i + 1] = g + p
                g = c * rr - bb
                if Z is not None:
                    zi, zj = Z[:, i].copy(), Z[:, i + 1].copy()
                    Z[:, i + 1] = s * zi + c * zj
                    Z[:, i] = c * zi - s * zj
                i -= 1
            if not hit_zero:
                d[l] -= p
                e[l] = g
                e[m] = 0.0
    darr = np.array(d)
    order = np.argsort(-darr, kind="stable")
    return darr[order], (Z[:, order] if Z is not None else None)


def signs_fixed(U, V):
    """Sign convention (linops.py:271-282): the largest-|.| entry of each
    v_j (first index on ties) is made positive, u_j flips along."""
    U = np.array(U, dtype=np.float64)
    V = np.array(V, dtype=np.float64)
    if V.shape[1] == 0:
        return U, V
    peak = V[np.argmax(np.abs(V), axis=0), np.arange(V.shape[1])]
    s = np.where(np.sign(peak) == 0, 1.0, np.sign(peak))
    return U * s, V * s


def _filter_columns(U):
    # CGS2 per column, cut at the first residual below 1e-2 (fsvd.py:145-155)
    U = U.copy()
    for j in range(U.shape[1]):
        v = _reorth(U[:, j], U[:, :j], 2)
        nv = float(np.linalg.norm(v))
        if nv < DEPENDENT_TOL:
            return U[:, :j], j
        U[:, j] = v / nv
    return U, U.shape[1]


@dataclass
class OraclePsvd:
    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    truncated: bool
    n_dropped: int
    gk: GKResult | None = None
    theta: np.ndarray | None = None


def fsvd_oracle(A, k, r, eps=1e-8, seed=0, reorth_passes=2, orthonormalize_u=True,
                start_mean=2.0, start_std=1.0, timings: dict | None = None) -> OraclePsvd:
    """Partial SVD (fsvd.py:158-204).  `timings` (optional) receives the
    wall seconds of the stages: gk, spectral, ritz_v (V = P G, n-sized) and
    ritz_u (the U products, filter and signs, m-sized)."""
    import time

    tick = time.perf_counter
    op = as_op(A)
    m, n = op.shape
    if not 1 <= r <= k <= min(m, n):
        raise OracleConfigError(f"need 1 <= r <= k <= min(m,n); got r={r}, k={k}")
    t0 = tick()
    g = gk_oracle(op, k, eps=eps, reorth_passes=reorth_passes, start_mean=start_mean,
                  start_std=start_std, seed=seed)
    t1 = tick()
    if g.degenerate:
        return OraclePsvd(np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0)), True, 0, g,
                          np.zeros(0))
    theta, G = ql_eig(*gram_of(g.alphas, g.betas))
    t2 = tick()
    top = math.sqrt(max(float(theta[0]), 0.0))
    keep = int(np.count_nonzero(theta > (DROP_REL * top) ** 2))
    take = min(r, keep)
    sig = np.sqrt(theta[:take])
    V = g.P @ G[:, :take]
    t3 = tick()
    U = np.empty((m, take))
    for j in range(take):  # the reference's `take` separate products
        U[:, j] = op.apply(V[:, j]) / sig[j]
    if orthonormalize_u and take:
        U, good = _filter_columns(U)
        if good < take:
            take, sig, V = good, sig[:good], V[:, :good]
    U, V = signs_fixed(U, V)
    if timings is not None:
        timings.update(gk=t1 - t0, spectral=t2 - t1, ritz_v=t3 - t2, ritz_u=tick() - t3)
    return OraclePsvd(U, sig, V, take < r, min(r, g.k_prime) - take, g, theta)


@dataclass
class OracleRank:
    rank: int
    k_prime: int
    eigenvalues: np.ndarray
    threshold: float
    mode: str
    gk: GKResult | None = None


def threshold_count(theta, eps, mode):
    """Strict count above eps (absolute) or eps^2 theta_1 (relative)
    (rank.py:33-48)."""
    if mode not in ("absolute", "relative"):
        raise OracleConfigError(f"mode {mode!r}")
    if not eps > 0:
        raise OracleConfigError("eps must be > 0")
    theta = np.asarray(theta, np.float64)
    if mode == "absolute":
        thr = float(eps)
    else:
        thr = float(eps) ** 2 * float(theta[0]) if theta.size else 0.0
    return int(np.count_nonzero(theta > thr)), thr


def rank_oracle(A, eps=1e-8, mode="absolute", seed=0, reorth_passes=2, gk_eps=1e-8,
                start_mean=2.0, start_std=1.0, k_max: int | None = None,
                timings: dict | None = None) -> OracleRank:
    """Numerical rank (rank.py:51-67): GK to min(m, n), eigenvalues without
    vectors, strict count.  `k_max` caps the loop below min(m, n) (timing
    samples only -- the reference always runs to min(m, n)); `timings`
    receives the stage seconds (gk, spectral)."""
    import time

    if mode not in ("absolute", "relative"):
        raise OracleConfigError(f"mode {mode!r}")
    if not eps > 0:
        raise OracleConfigError("eps must be > 0")
    op = as_op(A)
    t0 = time.perf_counter()
    g = gk_oracle(op, min(op.shape) if k_max is None else k_max, eps=gk_eps,
                  reorth_passes=reorth_passes, start_mean=start_mean, start_std=start_std,
                  seed=seed)
    t1 = time.perf_counter()
    if g.degenerate:
        return OracleRank(0, 0, np.zeros(0), eps if mode == "absolute" else 0.0, mode, g)
    theta, _ = ql_eig(*gram_of(g.alphas, g.betas), vectors=False)
    cnt, thr = threshold_count(theta, eps, mode)
    if timings is not None:
        timings.update(gk=t1 - t0, spectral=time.perf_counter() - t1)
    return OracleRank(cnt, g.k_prime, theta, thr, mode, g)
