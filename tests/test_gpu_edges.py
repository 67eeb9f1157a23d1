"""Edge cases of the CUDA path against the CPU oracle: extreme shapes, k_max
= 1, one reorthogonalization pass, immediate breakdown, wide vs tall, f32
storage, non-finite input, repeated calls on a resident matrix."""

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
from tests.parity import (COS_TOL_F64, SIG_RTOL_F64, assert_gk_match, col_cos, ortho_dev,
                          recurrence_dev, sig_relerr)

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1), (1, 7), (7, 1), (2, 2), (3, 17), (17, 3), (33, 65), (65, 33), (129, 257),
          (1000, 31), (31, 1000), (4097, 63), (63, 4097)]


@pytest.mark.parametrize("m,n", SHAPES)
def test_bidiag_shapes_vs_oracle(m, n):
    A = synth.gaussian_matrix(m, n, seed=m * 131 + n)
    k = min(m, n)
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=k, seed=3))
    ref = O.gk_oracle(A, k, seed=3)
    assert (st.k_prime, st.terminated_early, st.degenerate) == \
        (ref.k_prime, ref.terminated_early, ref.degenerate), (m, n)
    assert st.Q.shape == ref.Q.shape and st.P.shape == ref.P.shape
    assert_gk_match(st.alphas, st.betas, st.k_prime, ref.alphas, ref.betas, ref.k_prime,
                    kp_slack=0, what=f"{m}x{n}")
    if st.k_prime:
        assert ortho_dev(st.Q) < 1e-10 and ortho_dev(st.P) < 1e-10
        assert recurrence_dev(A, st.alphas, st.betas, st.Q, st.P) < 1e-10


@pytest.mark.parametrize("m,n", [(1, 1), (5, 3), (3, 5), (200, 40), (40, 200)])
def test_fsvd_shapes_vs_oracle(m, n):
    A = synth.gaussian_matrix(m, n, seed=7 + m + n)
    k = min(m, n)
    r = max(1, k // 2)
    ours = K.fsvd(A, k=k, r=r, cfg=K.BidiagConfig(k_max=k, seed=5))
    ref = O.fsvd_oracle(A, k, r, seed=5)
    assert ours.sigma.shape == ref.sigma.shape
    assert sig_relerr(ours.sigma, ref.sigma) <= SIG_RTOL_F64
    assert np.min(col_cos(ours.U, ref.U)) >= 1 - COS_TOL_F64
    assert np.min(col_cos(ours.V, ref.V)) >= 1 - COS_TOL_F64
    assert (ours.truncated, ours.n_dropped) == (ref.truncated, ref.n_dropped)


def test_k_max_one_and_single_pass_reorth():
    A = synth.low_rank_synth(300, 200, 30, seed=4)
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=1, seed=4))
    ref = O.gk_oracle(A, 1, seed=4)
    assert st.k_prime == 1 and st.Q.shape == (300, 2) and st.P.shape == (200, 1)
    assert abs(st.alphas[0] - ref.alphas[0]) <= 1e-12 * ref.alphas[0]
    assert abs(st.betas[1] - ref.betas[1]) <= 1e-12 * ref.betas[1]
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=100, reorth_passes=1, seed=4))
    ref = O.gk_oracle(A, 100, reorth_passes=1, seed=4)
    assert_gk_match(st.alphas, st.betas, st.k_prime, ref.alphas, ref.betas, ref.k_prime)
    assert ortho_dev(st.Q) < 1e-8


def test_large_eps_breaks_down_immediately():
    A = synth.gaussian_matrix(50, 40, seed=1)
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=40, eps=1e6, seed=1))
    ref = O.gk_oracle(A, 40, eps=1e6, seed=1)
    assert st.degenerate == ref.degenerate and st.k_prime == ref.k_prime == 0
    # eps between alpha_1 and beta_2: first beta breaks down, terminal column
    a1 = ref_a1 = O.gk_oracle(A, 1, seed=1).alphas[0]
    eps = 0.5 * min(a1, O.gk_oracle(A, 1, seed=1).betas[1])
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=40, eps=eps, seed=1))
    ref = O.gk_oracle(A, 40, eps=eps, seed=1)
    assert st.k_prime == ref.k_prime
    del ref_a1


def test_rank_shapes_and_modes():
    for m, n, l in [(1, 1, 1), (60, 20, 5), (20, 60, 5), (500, 400, 80)]:
        A = synth.low_rank_synth(m, n, l, seed=m + n)
        for eps, mode in [(1e-8, "absolute"), (1e-6, "relative")]:
            ours = K.estimate_rank(A, eps=eps, mode=mode)
            ref = O.rank_oracle(A, eps=eps, mode=mode)
            assert ours.rank == ref.rank == l, (m, n, l, mode)
            assert ours.threshold == pytest.approx(ref.threshold, rel=1e-10)


def test_float32_inputs_everywhere():
    A = synth.low_rank_synth(700, 300, 25, seed=6).astype(np.float32)
    A64 = A.astype(np.float64)
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=40, seed=6))
    ref = O.gk_oracle(A64, 40, seed=6)
    assert_gk_match(st.alphas, st.betas, st.k_prime, ref.alphas, ref.betas, ref.k_prime)
    assert K.estimate_rank(A).rank == O.rank_oracle(A64).rank == 25
    op = K.DeviceMatrix.from_host(A)
    assert op.dtype == np.float32
    assert np.array_equal(op.to_dense(), A)


def test_resident_matrix_reuse_is_deterministic():
    A = synth.low_rank_synth(3000, 900, 60, seed=8)
    op = K.DeviceMatrix.from_host(A)
    outs = [K.fsvd(op, k=90, r=20, cfg=K.BidiagConfig(k_max=90, seed=8)) for _ in range(3)]
    for o in outs[1:]:
        assert np.array_equal(o.sigma, outs[0].sigma)
        assert np.array_equal(o.U, outs[0].U) and np.array_equal(o.V, outs[0].V)
    reps = [K.estimate_rank(op) for _ in range(3)]
    for r_ in reps[1:]:
        assert np.array_equal(r_.eigenvalues, reps[0].eigenvalues)


def test_strided_and_noncontiguous_inputs():
    big = synth.gaussian_matrix(200, 150, seed=9)
    A = big[10:170:2, 5:125]  # strided rows, offset columns
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=40, seed=9))
    ref = O.gk_oracle(np.ascontiguousarray(A), 40, seed=9)
    assert_gk_match(st.alphas, st.betas, st.k_prime, ref.alphas, ref.betas, ref.k_prime)
    At = np.asfortranarray(synth.gaussian_matrix(90, 70, seed=10))
    assert K.estimate_rank(At).rank == O.rank_oracle(np.ascontiguousarray(At)).rank


def test_nan_and_inf_raise_numerical_error():
    for bad in (np.nan, np.inf, -np.inf):
        A = synth.gaussian_matrix(64, 48, seed=2)
        A[17, 33] = bad
        with pytest.raises(K.NumericalError):
            K.estimate_rank(A)


def test_golden_and_edges_through_streaming_kernels():
    """The reference-generated golden cases (breakdowns, degenerate and
    terminal columns included), this module's edge cases and the restart
    suite with the
    whole-loop resident kernel disabled (KSVD_RESIDENT=0): the small shapes
    then run the streaming kernels -- the paired step (k_cgs2_pair, pair.cuh)
    wherever its tiles fit -- in a subprocess (the switch is read once)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    here = Path(__file__).resolve()
    par = root / "tests" / "test_gpu_parity.py"
    ids = [f"{par}::{t}" for t in ("test_bidiag_golden", "test_fsvd_golden", "test_rank_golden",
                                   "test_bidiag_edge_cases", "test_nonfinite_raises",
                                   "test_spurious_filter_stops_at_rank")]
    ids += [f"{here}::{t}" for t in ("test_bidiag_shapes_vs_oracle", "test_fsvd_shapes_vs_oracle",
                                     "test_k_max_one_and_single_pass_reorth",
                                     "test_large_eps_breaks_down_immediately",
                                     "test_rank_shapes_and_modes", "test_float32_inputs_everywhere",
                                     "test_nan_and_inf_raise_numerical_error")]
    rst = root / "tests" / "test_gpu_restart.py"  # thick restarts resume through the paired step
    ids += [f"{rst}::{t}" for t in ("test_restarted_matches_oracle_and_dense_svd",
                                    "test_restart_beats_plain_fsvd_at_equal_basis_size",
                                    "test_restarted_low_rank_f32_and_factored",
                                    "test_restarted_full_basis_and_errors",
                                    "test_breakdown_residual_reported_not_zeroed")]
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          *ids], cwd=root, env={**os.environ, "KSVD_RESIDENT": "0"},
                         capture_output=True, text=True, timeout=1200)
    assert res.returncode == 0, res.stdout[-3000:]
