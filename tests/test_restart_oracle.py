"""The restarted-mode CPU restatement (oracle/restarted.py) against a dense
SVD: converged triplets are basis-independent, so this pins the restatement
without a reference counterpart (restarts are a non-goal of the reference,
SPEC.md:155)."""

import numpy as np
import pytest

from oracle.restarted import restarted_oracle
from paper_2104_10785_b200 import synth


def _spectrum_matrix(m, n, decay, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
    V, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
    s = decay ** np.arange(min(m, n))
    return (U * s) @ V.T, s


@pytest.mark.parametrize("m,n,r,k", [(300, 200, 5, 15), (200, 300, 8, 20), (400, 120, 3, 10)])
def test_restarted_oracle_converges_to_dense_svd(m, n, r, k):
    A, s = _spectrum_matrix(m, n, 0.93, seed=m + n)
    U, sig, V, restarts, resid = restarted_oracle(A, r, k, tol=1e-12, seed=1)
    assert restarts >= 1  # k too small to converge in one cycle
    assert np.allclose(sig, s[:r], rtol=1e-10)
    assert np.all(resid <= 1e-12 * sig[0])
    assert np.allclose(A @ V, U * sig, atol=1e-9 * sig[0])
    assert np.allclose(A.T @ U, V * sig, atol=1e-9 * sig[0])
    assert np.allclose(U.T @ U, np.eye(r), atol=1e-10)


def test_restarted_oracle_exact_low_rank_stops_early():
    A = synth.low_rank_synth(150, 100, 6, seed=2)
    U, sig, V, restarts, resid = restarted_oracle(A, 4, 12, seed=3)
    ref = np.linalg.svd(A, compute_uv=False)[:4]
    assert restarts == 0 and np.allclose(sig, ref, rtol=1e-12)
