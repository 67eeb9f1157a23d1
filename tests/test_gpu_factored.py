"""FactoredOperator (reference linops.py:176-205) on the device: products
against the formed matrix, and the GK path (bidiagonalize / fsvd /
estimate_rank) on a factored operator against the oracle run on the formed
matrix -- including the retraction caller's shifted-operator shape
(manifold.py:121-130: left [U, Up], 2r x 2r core, right [V, Vp])."""

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from tests.parity import (COS_TOL_F64, SIG_RTOL_F64, assert_gk_match, col_cos, ortho_dev,
                          recurrence_dev, sig_relerr)

pytestmark = pytest.mark.gpu


def _factors(d1, d2, s1, s2, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((d1, s1)), rng.standard_normal((s1, s2)),
            rng.standard_normal((d2, s2)))


def _shifted(d1, d2, r, step, seed):
    """W + step * xi in the factored form the retraction builds."""
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((d1, r)))
    V, _ = np.linalg.qr(rng.standard_normal((d2, r)))
    S = np.sort(rng.uniform(1.0, 10.0, r))[::-1]
    Up = rng.standard_normal((d1, r))
    Up -= U @ (U.T @ Up)
    Vp = rng.standard_normal((d2, r))
    Vp -= V @ (V.T @ Vp)
    Mc = rng.standard_normal((r, r))
    core = np.zeros((2 * r, 2 * r))
    core[:r, :r] = np.diag(S) + step * Mc
    core[:r, r:] = step * np.eye(r)
    core[r:, :r] = step * np.eye(r)
    return np.hstack([U, Up]), core, np.hstack([V, Vp])


@pytest.mark.parametrize("d1,d2,s1,s2", [(1, 1, 1, 1), (50, 30, 4, 4), (300, 1000, 7, 3),
                                         (4097, 129, 20, 20), (1000, 20000, 12, 40)])
def test_products_match_formed_matrix(d1, d2, s1, s2):
    L, Cc, R = _factors(d1, d2, s1, s2, seed=d1 + d2)
    op = K.FactoredOperator(L, Cc, R)
    A = L @ Cc @ R.T
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(d2), rng.standard_normal(d1)
    tol = 1e-12 * np.sqrt(d1 + d2) * max(1.0, np.abs(A).max())
    assert op.shape == (d1, d2)
    assert np.allclose(op.matvec(x), A @ x, rtol=1e-12, atol=tol * np.abs(x).sum())
    assert np.allclose(op.rmatvec(y), A.T @ y, rtol=1e-12, atol=tol * np.abs(y).sum())
    X = rng.standard_normal((d2, 3))
    assert np.allclose(op.matmat(X), A @ X, rtol=1e-12, atol=tol * np.abs(X).sum())
    if d1 * d2 <= 1_000_000:
        assert np.allclose(op.to_dense(), A, rtol=1e-12, atol=1e-12 * np.abs(A).max())


def test_fsvd_and_rank_on_shifted_operator():
    left, core, right = _shifted(3000, 2000, 8, -0.3, seed=4)
    op = K.FactoredOperator(left, core, right)
    A = left @ core @ right.T
    for k, r in [(16, 8), (12, 5)]:
        ours = K.fsvd(op, k=k, r=r, cfg=K.BidiagConfig(k_max=k, seed=7))
        ref = O.fsvd_oracle(A, k, r, seed=7)
        assert ours.sigma.shape == ref.sigma.shape
        assert sig_relerr(ours.sigma, ref.sigma) <= SIG_RTOL_F64
        assert np.min(col_cos(ours.U, ref.U)) >= 1 - COS_TOL_F64
        assert np.min(col_cos(ours.V, ref.V)) >= 1 - COS_TOL_F64
    rep = K.estimate_rank(op)
    assert rep.rank == O.rank_oracle(A).rank == 16


def test_bidiagonalize_on_factored_operator():
    L, Cc, R = _factors(700, 500, 30, 25, seed=11)
    op = K.FactoredOperator(L, Cc, R)
    A = L @ Cc @ R.T
    st = K.bidiagonalize(op, K.BidiagConfig(k_max=40, seed=3))
    ref = O.gk_oracle(A, 40, seed=3)
    assert_gk_match(st.alphas, st.betas, st.k_prime, ref.alphas, ref.betas, ref.k_prime)
    # rank 25: k' lands at 25-26 (past the rank the step is rounding noise,
    # SURVEY.md 8(c) probe 5), always with an early stop
    assert st.terminated_early and 25 <= st.k_prime <= 27 and abs(st.k_prime - ref.k_prime) <= 2
    assert ortho_dev(st.P) < 1e-10 and ortho_dev(st.Q[:, :25]) < 1e-10
    assert recurrence_dev(A, st.alphas, st.betas, st.Q, st.P) < 1e-10


def test_factored_has_no_dense_rows_through_the_abi(tmp_path):
    op = K.FactoredOperator(*_factors(20, 10, 3, 3, seed=1))
    with pytest.raises(K.ConfigError):
        K.write_matrix_device(tmp_path / "f.klrm", op)
    with pytest.raises(K.NumericalError):
        L, Cc, R = _factors(40, 30, 4, 4, seed=2)
        Cc[1, 2] = np.nan
        K.estimate_rank(K.FactoredOperator(L, Cc, R))


_NCCL_SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r})
import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from tests.parity import col_cos, sig_relerr
rng = np.random.default_rng(5)
L, Cc, R = rng.standard_normal((2000, 10)), rng.standard_normal((10, 10)), rng.standard_normal((900, 10))
A = L @ Cc @ R.T
ours = K.fsvd(K.FactoredOperator(L, Cc, R), k=14, r=6, cfg=K.BidiagConfig(k_max=14, seed=2))
ref = O.fsvd_oracle(A, 14, 6, seed=2)
print(json.dumps([sig_relerr(ours.sigma, ref.sigma), float(np.min(col_cos(ours.U, ref.U))),
                  K.estimate_rank(K.FactoredOperator(L, Cc, R)).rank]))
"""


def test_factored_multi_rank_code_path():
    """KSVD_FORCE_NCCL: the multi-rank path (L^T q all-reduced over NCCL,
    multi-kernel CGS) on a 1-rank communicator."""
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
    rel, cos, rank = json.loads(res.stdout.strip().splitlines()[-1])
    assert rel <= SIG_RTOL_F64 and cos >= 1 - COS_TOL_F64 and rank == 10


def test_reference_style_factored_object_is_accelerated():
    """An object shaped like the reference's FactoredOperator (left, core,
    right, matvec) passed to fsvd runs on the device from its factors."""

    class RefFactored:  # stand-in for krysvd.linops.FactoredOperator
        def __init__(self, left, core, right):
            self.left, self.core, self.right = left, core, right
            self.shape = (left.shape[0], right.shape[0])

        def matvec(self, x):
            raise AssertionError("host product called")

        rmatvec = matvec

    L, Cc, R = _factors(800, 600, 9, 9, seed=21)
    ours = K.fsvd(RefFactored(L, Cc, R), k=12, r=4, cfg=K.BidiagConfig(k_max=12, seed=1))
    ref = O.fsvd_oracle(L @ Cc @ R.T, 12, 4, seed=1)
    assert sig_relerr(ours.sigma, ref.sigma) <= SIG_RTOL_F64
