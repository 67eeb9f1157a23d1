"""Restarted GK (opt-in, beyond the reference) on the
device against its CPU restatement (oracle/restarted.py) and the dense
SVD."""

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle.restarted import restarted_oracle
from paper_2104_10785_b200 import synth
from tests.parity import col_cos

pytestmark = pytest.mark.gpu


def _spectrum_matrix(m, n, decay, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
    V, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
    s = decay ** np.arange(min(m, n))
    return (U * s) @ V.T, s


@pytest.mark.parametrize("m,n,r,k", [(300, 200, 5, 15), (200, 300, 8, 20), (400, 120, 3, 10),
                                     (3000, 1500, 10, 30)])
def test_restarted_matches_oracle_and_dense_svd(m, n, r, k):
    A, s = _spectrum_matrix(m, n, 0.93, seed=m + n)
    cfg = K.BidiagConfig(k_max=k, seed=1)
    ps, info = K.fsvd_restarted(A, r, k=k, tol=1e-12, cfg=cfg)
    U, sig, V, restarts, resid = restarted_oracle(A, r, k, tol=1e-12, seed=1)
    assert info.converged and info.restarts >= 1
    assert abs(info.restarts - restarts) <= 1
    assert np.allclose(ps.sigma, s[:r], rtol=1e-10)
    assert np.allclose(ps.sigma, sig, rtol=1e-10)
    assert np.min(col_cos(ps.U, U)) >= 1 - 1e-8 and np.min(col_cos(ps.V, V)) >= 1 - 1e-8
    assert np.allclose(A @ ps.V, ps.U * ps.sigma, atol=1e-9 * ps.sigma[0])
    assert np.allclose(A.T @ ps.U, ps.V * ps.sigma, atol=1e-9 * ps.sigma[0])
    assert np.all(info.residuals <= 1e-12 * ps.sigma[0])
    # sign convention of fix_signs (linops.py:271-282) on V
    lead = ps.V[np.argmax(np.abs(ps.V), axis=0), np.arange(r)]
    assert np.all(lead > 0)


def test_restart_beats_plain_fsvd_at_equal_basis_size():
    """Same k: plain fsvd is not converged (SURVEY 8(c) probe 6), the
    restarted mode is."""
    A, s = _spectrum_matrix(2000, 1000, 0.97, seed=5)
    plain = K.fsvd(A, k=30, r=10, cfg=K.BidiagConfig(k_max=30, seed=0))
    ps, info = K.fsvd_restarted(A, 10, k=30, tol=1e-12, cfg=K.BidiagConfig(k_max=30, seed=0))
    err_plain = np.max(np.abs(plain.sigma - s[:10]) / s[:10])
    err_rest = np.max(np.abs(ps.sigma - s[:10]) / s[:10])
    assert err_rest <= 1e-10 < err_plain


def test_restarted_low_rank_f32_and_factored():
    A = synth.low_rank_synth(500, 300, 6, seed=2)
    ref = np.linalg.svd(A, compute_uv=False)
    ps, info = K.fsvd_restarted(A, 4, k=12, cfg=K.BidiagConfig(k_max=12, seed=3))
    assert info.restarts == 0 and info.converged and np.allclose(ps.sigma, ref[:4], rtol=1e-12)
    A32 = _spectrum_matrix(800, 400, 0.9, seed=8)[0].astype(np.float32)
    ref32 = np.linalg.svd(A32.astype(np.float64), compute_uv=False)
    ps, info = K.fsvd_restarted(A32, 6, k=16, tol=1e-11)
    assert info.converged and np.allclose(ps.sigma, ref32[:6], rtol=1e-9)
    rng = np.random.default_rng(4)
    L, Cc, R = rng.standard_normal((900, 40)), np.diag(0.9 ** np.arange(40)), \
        rng.standard_normal((700, 40))
    Af = L @ Cc @ R.T
    ps, info = K.fsvd_restarted(K.FactoredOperator(L, Cc, R), 5, k=14, tol=1e-12)
    assert info.converged and info.restarts >= 1
    assert np.allclose(ps.sigma, np.linalg.svd(Af, compute_uv=False)[:5], rtol=1e-10)


def test_restarted_full_basis_and_errors():
    A, s = _spectrum_matrix(60, 40, 0.8, seed=1)
    ps, info = K.fsvd_restarted(A, 5, k=40)
    assert info.restarts == 0 and np.allclose(ps.sigma, s[:5], rtol=1e-10)
    for bad in (dict(r=0), dict(r=5, k=4), dict(r=5, k=41), dict(r=5, k=10, keep=10),
                dict(r=5, k=10, tol=0.0)):
        with pytest.raises(K.ConfigError):
            K.fsvd_restarted(A, **bad)


_NCCL_SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r})
import paper_2104_10785_b200 as K
rng = np.random.default_rng(3)
U, _ = np.linalg.qr(rng.standard_normal((1500, 400)))
V, _ = np.linalg.qr(rng.standard_normal((400, 400)))
s = 0.95 ** np.arange(400)
A = (U * s) @ V.T
ps, info = K.fsvd_restarted(A, 6, k=18, tol=1e-12)
print(json.dumps([float(np.max(np.abs(ps.sigma - s[:6]) / s[:6])), info.restarts, info.converged]))
"""


def test_restarted_multi_rank_code_path():
    """KSVD_FORCE_NCCL: restart on the multi-rank path (NCCL all-reduces,
    multi-kernel CGS) over a 1-rank communicator."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parent.parent)
    res = subprocess.run([sys.executable, "-c", _NCCL_SCRIPT.format(root=root)],
                         env={**os.environ, "KSVD_FORCE_NCCL": "1"}, capture_output=True,
                         text=True, timeout=600, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    err, restarts, conv = json.loads(res.stdout.strip().splitlines()[-1])
    assert err <= 1e-10 and restarts >= 1 and conv


def test_dense_svd_single_cta_kernel():
    """k_dense_svd_cta (ksvd_dense_svd_dev) against LAPACK, incl. odd k (the
    dummy round-robin player), exact zero singular values and the host
    fallback above the shared-memory limit."""
    from paper_2104_10785_b200 import _lib
    from paper_2104_10785_b200.restart import dense_svd
    ctx = _lib.get_context()
    rng = np.random.default_rng(11)
    for k in (1, 2, 7, 30, 31, 64, 101, 130):
        T = np.triu(rng.standard_normal((k, k)))
        if k > 5:
            T[-1, :] = 0.0  # a zero singular value (an alpha breakdown's T)
        Uh, s, Vh = dense_svd(T, ctx)
        ref = np.linalg.svd(T, compute_uv=False)
        assert np.allclose(s, ref, rtol=1e-12, atol=1e-14 * ref[0]), k
        assert np.allclose((Uh * s) @ Vh.T, T, atol=1e-12 * ref[0]), k
        assert np.allclose(Vh.T @ Vh, np.eye(k), atol=1e-12), k
        assert np.all(np.diff(s) <= 0)


def test_breakdown_residual_reported_not_zeroed():
    """A GK breakdown (beta_{k'+1} < eps, ABSOLUTE 1e-8) is not convergence
    at a tighter tol: the residuals come from the breakdown scalar and the
    same tol test decides `converged`.  A = rank 6 + 1e-10 noise
    breaks down after 7 steps; the 7th Ritz triplet sits at the noise level
    with a residual of the order of beta_8 -- far above tol * s_1."""
    A = synth.low_rank_synth(500, 300, 6, seed=2)
    A = A + 1e-10 * np.random.default_rng(5).standard_normal(A.shape)
    tol = 1e-14
    ps, info = K.fsvd_restarted(A, 7, k=12, tol=tol, cfg=K.BidiagConfig(k_max=12, seed=3))
    assert info.k_prime < 12 and ps.sigma.shape[0] == 7  # broke down early
    true_res = np.linalg.norm(A @ ps.V - ps.U * ps.sigma, axis=0)
    assert np.all(info.residuals > 0)
    assert info.converged == bool(np.all(info.residuals <= tol * ps.sigma[0]))
    assert not info.converged and info.residuals[-1] > tol * ps.sigma[0]
    np.testing.assert_allclose(true_res, info.residuals, rtol=0.05, atol=1e-13 * ps.sigma[0])
