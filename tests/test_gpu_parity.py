"""Parity of the CUDA path (through the C ABI) with the reference.

Two checkers: the golden vectors the reference produced
(tests/golden/make_golden.py) and the CPU oracle run here on the same
seeded inputs.  Tolerances are the north star's (tests/parity.py): fp64
sigma relative error <= 1e-10, |cos| >= 1 - 1e-8; fp32 storage relative
error <= 1e-4 and residual <= 1e-4 sigma_1; ranks exact.
"""

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
from tests.conftest import golden_cases
from tests.golden.recipes import build_input
from tests.parity import (COS_TOL_F64, RES_TOL_F32, SIG_RTOL_F32, SIG_RTOL_F64,
                          assert_gk_match, col_cos, ortho_dev, recurrence_dev,
                          sig_relerr)

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- products
@pytest.mark.parametrize("m,n", [(1, 1), (7, 5), (50, 30), (300, 1000), (2049, 129),
                                 (4000, 9001), (1000, 20000)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_matvec_rmatvec(m, n, dtype):
    rng = np.random.default_rng(m * 7 + n)
    A = rng.standard_normal((m, n)).astype(dtype)
    op = K.DeviceMatrix.from_host(A)
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    A64 = A.astype(np.float64)
    ref_y, ref_z = A64 @ x, A64.T @ y
    tol = 1e-12 * np.sqrt(n)
    assert np.allclose(op.matvec(x), ref_y, rtol=tol, atol=tol * np.abs(ref_y).max())
    assert np.allclose(op.rmatvec(y), ref_z, rtol=tol, atol=tol * np.abs(ref_z).max())
    X = rng.standard_normal((n, 3))
    assert np.allclose(op.matmat(X), A64 @ X, rtol=tol, atol=tol * np.abs(A64 @ X).max())
    assert np.array_equal(op.to_dense(), A)


def test_adjoint_identity():
    rng = np.random.default_rng(5)
    for m, n in [(3, 8), (64, 17), (513, 1025)]:
        A = rng.standard_normal((m, n))
        op = K.DeviceMatrix.from_host(A)
        x, y = rng.standard_normal(n), rng.standard_normal(m)
        lhs, rhs = float(op.matvec(x) @ y), float(x @ op.rmatvec(y))
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs), abs(rhs))


def test_products_deterministic():
    rng = np.random.default_rng(9)
    A = rng.standard_normal((3000, 2500))
    op = K.DeviceMatrix.from_host(A)
    x, y = rng.standard_normal(2500), rng.standard_normal(3000)
    assert np.array_equal(op.matvec(x), op.matvec(x))
    assert np.array_equal(op.rmatvec(y), op.rmatvec(y))


# ---------------------------------------------------------------- GK loop
def test_bidiag_golden(golden):
    for parts in golden_cases(golden, "bidiag"):
        key, recipe, k, seed, reorth = parts[0], parts[1], int(parts[2]), int(parts[3]), int(parts[4])
        A = build_input(recipe)
        st = K.bidiagonalize(A, K.BidiagConfig(k_max=k, seed=seed, reorth_passes=reorth))
        info = golden[key + "/info"]
        assert [int(st.terminated_early), int(st.degenerate)] == list(info[1:3]), (recipe, info)
        assert st.Q.shape[1] - st.k_prime == info[3] - info[0], (recipe, info)
        assert_gk_match(st.alphas, st.betas, st.k_prime, golden[key + "/alphas"],
                        golden[key + "/betas"], info[0], what=recipe)
        if key + "/Q" in golden and st.k_prime:
            h = min(8, st.k_prime)
            assert np.min(col_cos(st.Q[:, :h], golden[key + "/Q"][:, :h])) >= 1 - COS_TOL_F64, recipe
            assert np.min(col_cos(st.P[:, :h], golden[key + "/P"][:, :h])) >= 1 - COS_TOL_F64, recipe
        if st.k_prime:
            tol = 1e-8 if reorth == 1 else 1e-10
            assert ortho_dev(st.Q) < tol, recipe
            assert ortho_dev(st.P) < 1e-10, recipe
            assert recurrence_dev(A, st.alphas, st.betas, st.Q, st.P) < 1e-10, recipe


def test_start_vector_pinned_bitwise(golden):
    A = synth.gaussian_matrix(8, 8, seed=1)
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=4, seed=42))
    assert np.array_equal(st.Q[:, 0], golden["start/42/8/2.0/1.0"])
    st = K.bidiagonalize(synth.gaussian_matrix(6, 6, seed=1),
                         K.BidiagConfig(k_max=3, start_mean=-1.0, start_std=0.5, seed=9))
    assert np.array_equal(st.Q[:, 0], golden["start/9/6/-1.0/0.5"])


def test_bidiag_edge_cases():
    st = K.bidiagonalize(np.zeros((6, 4)), K.BidiagConfig(k_max=4, seed=3))
    assert st.degenerate and st.k_prime == 0 and st.terminated_early
    assert st.alphas.shape == (0,) and st.betas.shape == (1,)
    assert st.Q.shape == (6, 1) and st.P.shape == (4, 0)
    st = K.bidiagonalize(np.eye(5), K.BidiagConfig(k_max=5, seed=7))
    assert st.k_prime == 1 and st.terminated_early and abs(st.alphas[0] - 1) < 1e-12
    assert st.betas[1] < 1e-8 and st.Q.shape == (5, 2) and ortho_dev(st.Q) < 1e-12
    assert np.allclose(st.P[:, 0], st.Q[:, 0], atol=1e-14)
    A = synth.gaussian_matrix(30, 30, seed=13)
    st = K.bidiagonalize(A, K.BidiagConfig(k_max=30, seed=13))
    assert st.k_prime == 30 and st.terminated_early and st.Q.shape == (30, 30)
    # 1 x n and m x 1
    st = K.bidiagonalize(np.arange(1.0, 6.0)[None, :], K.BidiagConfig(k_max=1, seed=0))
    assert st.k_prime == 1 and abs(st.alphas[0] - np.sqrt(55.0)) < 1e-12


def test_bidiag_determinism():
    A = synth.low_rank_synth(80, 60, 20, seed=31)
    cfg = K.BidiagConfig(k_max=40, seed=31)
    a, b = K.bidiagonalize(A, cfg), K.bidiagonalize(A, cfg)
    for f in ("alphas", "betas", "Q", "P"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert not np.array_equal(a.Q[:, 0], K.bidiagonalize(A, K.BidiagConfig(k_max=40, seed=2)).Q[:, 0])


def test_nonfinite_raises():
    A = synth.gaussian_matrix(20, 10, seed=1)
    A[3, 4] = np.nan
    with pytest.raises(K.NumericalError):
        K.bidiagonalize(A, K.BidiagConfig(k_max=5))
    A = synth.gaussian_matrix(20, 10, seed=1)
    A[7, 2] = np.inf
    with pytest.raises(K.NumericalError):
        K.fsvd(A, k=5, r=2)


def test_config_errors_on_device():
    op = K.DeviceMatrix.from_host(np.eye(4))
    with pytest.raises(K.ConfigError):
        K.run_gk(op, K.BidiagConfig(k_max=5))
    with pytest.raises(K.ConfigError):
        K.as_operator(type("Op", (K.LinearOperator,), {"shape": (3, 3)})())


# ---------------------------------------------------------------- fsvd
def test_fsvd_golden(golden):
    for parts in golden_cases(golden, "fsvd"):
        key, recipe = parts[0], parts[1]
        k, r, seed, eps, ortho = int(parts[2]), int(parts[3]), int(parts[4]), float(parts[5]), \
            bool(int(parts[6]))
        A = build_input(recipe)
        psvd, st, theta = K.fsvd(A, k=k, r=r, cfg=K.BidiagConfig(k_max=k, seed=seed, eps=eps),
                                 orthonormalize_u=ortho, return_details=True)
        info = golden[key + "/info"]
        assert [int(psvd.truncated), psvd.n_dropped, st.k_prime, psvd.sigma.shape[0]] == \
            list(info), (recipe, info)
        assert sig_relerr(psvd.sigma, golden[key + "/sigma"]) <= SIG_RTOL_F64, recipe
        nk = golden[key + "/U"].shape[1]
        if nk:
            assert np.min(col_cos(psvd.U[:, :nk], golden[key + "/U"])) >= 1 - COS_TOL_F64, recipe
            assert np.min(col_cos(psvd.V[:, :nk], golden[key + "/V"])) >= 1 - COS_TOL_F64, recipe
            # identical sign convention (fix_signs on the device)
            assert np.allclose(psvd.V[:, :nk], golden[key + "/V"], atol=1e-7), recipe
            assert np.allclose(psvd.U[:, :nk], golden[key + "/U"], atol=1e-7), recipe


def test_fsvd_vs_oracle_config1():
    A = synth.config1_matrix(seed=0)
    ours = K.fsvd(A, k=30, r=10, cfg=K.BidiagConfig(k_max=30, eps=1e-10, seed=0))
    ref = O.fsvd_oracle(A, 30, 10, eps=1e-10, seed=0)
    assert sig_relerr(ours.sigma, ref.sigma) <= SIG_RTOL_F64
    assert np.min(col_cos(ours.U, ref.U)) >= 1 - COS_TOL_F64
    assert np.min(col_cos(ours.V, ref.V)) >= 1 - COS_TOL_F64


def test_fsvd_float32_storage():
    rng = np.random.default_rng(4)
    m, n, r = 3000, 1200, 40
    P, _ = np.linalg.qr(rng.standard_normal((m, r)))
    Q, _ = np.linalg.qr(rng.standard_normal((n, r)))
    s = 100.0 * np.exp(-np.arange(1, r + 1) / 20.0)
    A32 = ((P * s) @ Q.T + 1e-4 * rng.standard_normal((m, n)) / np.sqrt(n)).astype(np.float32)
    ours = K.fsvd(A32, k=96, r=32, cfg=K.BidiagConfig(k_max=96, seed=3))
    ref = O.fsvd_oracle(A32.astype(np.float64), 96, 32, seed=3)
    assert sig_relerr(ours.sigma, ref.sigma) <= SIG_RTOL_F32
    A64 = A32.astype(np.float64)
    res = np.linalg.norm(A64 @ ours.V - ours.U * ours.sigma, axis=0)
    assert np.max(res) <= RES_TOL_F32 * ours.sigma[0]
    # f32 storage with f64 accumulation is in fact fp64-accurate
    assert sig_relerr(ours.sigma, ref.sigma) <= 1e-10


def test_fsvd_properties():
    A = synth.low_rank_synth(100, 80, 40, seed=3)
    psvd, state, theta = K.fsvd(A, k=20, r=20, cfg=K.BidiagConfig(k_max=20, seed=3),
                                return_details=True)
    assert state.k_prime == 20 and not state.terminated_early
    theta2, _ = K.symtridiag_eig(K.gram_tridiag(state))
    assert np.array_equal(theta, theta2)
    a = K.fsvd(A, k=30, r=12, cfg=K.BidiagConfig(k_max=30, seed=10))
    b = K.fsvd(A, k=30, r=12, cfg=K.BidiagConfig(k_max=30, seed=10))
    assert np.array_equal(a.sigma, b.sigma) and np.array_equal(a.U, b.U)
    assert np.array_equal(a.V, b.V)


def test_spurious_filter_stops_at_rank():
    A = synth.low_rank_synth(1000, 1000, 100, seed=5)
    psvd = K.fsvd(A, k=1000, r=1000)
    assert psvd.sigma.shape[0] == 100
    assert ortho_dev(psvd.U) < 1e-10 and ortho_dev(psvd.V) < 1e-10
    R = A - (psvd.U * psvd.sigma) @ psvd.V.T
    assert np.linalg.norm(R) / np.linalg.norm(A) < 1e-12


# ---------------------------------------------------------------- rank
def test_rank_golden(golden):
    for parts in golden_cases(golden, "rank"):
        key, recipe, eps, mode, seed = parts[0], parts[1], float(parts[2]), parts[3], int(parts[4])
        A = build_input(recipe)
        rep = K.estimate_rank(A, eps=eps, mode=mode, cfg=K.BidiagConfig(k_max=1, seed=seed))
        rank_ref, kp_ref = golden[key + "/info"]
        assert rep.rank == rank_ref, recipe  # bit-exact
        assert abs(rep.k_prime - kp_ref) <= 2, (recipe, rep.k_prime, kp_ref)
        ev = golden[key + "/eigenvalues"]
        n = min(rep.rank, ev.size)
        if n:
            assert sig_relerr(rep.eigenvalues[:n], ev[:n]) <= SIG_RTOL_F64, recipe
        assert rep.mode == mode


@pytest.mark.slow
def test_rank_config2_exact():
    A = synth.config2_matrix(seed=1)
    rep = K.estimate_rank(A, eps=1e-6, mode="relative", cfg=K.BidiagConfig(k_max=1, seed=1))
    ref = O.rank_oracle(A, eps=1e-6, mode="relative", seed=1)
    assert rep.rank == ref.rank == 137
    assert sig_relerr(rep.eigenvalues[:137], ref.eigenvalues[:137]) <= SIG_RTOL_F64


def test_rank_scale_invariant_and_monotone():
    A = synth.low_rank_synth(50, 40, 10, seed=8)
    r1 = K.estimate_rank(A, eps=1e-6, mode="relative")
    r2 = K.estimate_rank(1e6 * A, eps=1e-6, mode="relative")
    assert r1.rank == r2.rank == 10 and r2.threshold > r1.threshold
    A = synth.low_rank_synth(60, 60, 12, seed=9)
    assert K.estimate_rank(A, eps=1e-2).rank <= K.estimate_rank(A, eps=1e-12).rank
    assert K.estimate_rank(A, eps=1e-8).rank == 12


def test_device_matrix_reuse_and_torch_input():
    torch = pytest.importorskip("torch")
    A = synth.low_rank_synth(400, 300, 30, seed=2)
    op = K.DeviceMatrix.from_host(A)
    r_np = K.estimate_rank(A)
    r_dev = K.estimate_rank(op)
    assert r_np.rank == r_dev.rank == 30
    t = torch.from_numpy(A).cuda()
    r_t = K.estimate_rank(t)
    assert r_t.rank == 30 and np.array_equal(r_t.eigenvalues, r_dev.eigenvalues)


# ---------------------------------------------------------------- CGS paths
_PATH_SCRIPT = r"""
import sys, json
sys.path.insert(0, {root!r})
import numpy as np
import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
out = []
for (m, n, l, k, seed) in [(300, 200, 40, 60, 6), (2000, 700, 120, 200, 3), (5000, 1200, 300, 400, 9)]:
    A = synth.low_rank_synth(m, n, l, seed=seed)
    ps = K.fsvd(A, k=k, r=min(l, 30), cfg=K.BidiagConfig(k_max=k, seed=seed))
    ref = O.fsvd_oracle(A, k, min(l, 30), seed=seed)
    rel = float(np.max(np.abs(ps.sigma - ref.sigma) / ref.sigma))
    cos = float(min(np.min(np.abs(np.einsum("ij,ij->j", ps.U, ref.U))),
                    np.min(np.abs(np.einsum("ij,ij->j", ps.V, ref.V)))))
    # relative threshold: absolute 1e-8 sits at the rounding level of the
    # post-rank Ritz values for these spectra (see tools/diag_paths.py)
    rep = K.estimate_rank(A, eps=1e-6, mode="relative", cfg=K.BidiagConfig(k_max=1, seed=seed))
    out.append([rel, cos, rep.rank, l])
print(json.dumps(out))
"""


_MULTI = {"KSVD_RESIDENT": "0"}  # small cases would otherwise take the resident kernel


@pytest.mark.parametrize("env", [{"KSVD_COOP": "0", **_MULTI},
                                 {"KSVD_FORCE_NCCL": "1"}, {"KSVD_FORCE_PX": "1"},
                                 {"KSVD_FORCE_NCCL": "1", "KSVD_MTILE": "0"},
                                 {"KSVD_FORCE_PX": "1", "KSVD_MTILE": "0"},
                                 {"KSVD_FORCE_NCCL": "1", "KSVD_PDL_MULTI": "0"},
                                 {"KSVD_FORCE_NCCL": "1", "KSVD_FORCE_COOP": "1"},
                                 {"KSVD_RED_MAX": "0", **_MULTI},
                                 {"KSVD_RED_MAX": "100000000", **_MULTI}, {"KSVD_PDL": "0", **_MULTI},
                                 {"KSVD_FORCE_COOP": "1", **_MULTI},
                                 {"KSVD_PAIR": "0", **_MULTI}, {"KSVD_TAILFIN": "0", **_MULTI},
                                 _MULTI, {}])
def test_cgs_paths_agree(env):
    """The whole-loop resident kernel (small matrices, default), the
    tile-resident k_cgs2_tile2 (redundant or distributed reductions) and the
    multi-kernel CGS2 path (KSVD_COOP=0) all meet the parity bar, with and
    without programmatic dependent launch, launched regularly with the flip
    grid barrier (default) or cooperatively (KSVD_FORCE_COOP: the fallback
    when the residency probe fails); KSVD_FORCE_NCCL runs the multi-rank code
    path (NCCL all-reduces between the kernels, k_cgs_tile_phase) over a
    1-rank communicator, KSVD_FORCE_PX the same path with every all-reduce
    through the NVLink peer-exchange kernel (csrc/peer.cuh) instead.
    _MULTI takes the paired step (both CGS2 in k_cgs2_pair, pair.cuh) where
    its tiles fit; KSVD_PAIR=0 the serialised step, KSVD_TAILFIN=0 the paired
    step with a separate w finalisation kernel."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parent.parent)
    res = subprocess.run([sys.executable, "-c", _PATH_SCRIPT.format(root=root)],
                         env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    for rel, cos, rank, l in json.loads(res.stdout.strip().splitlines()[-1]):
        assert rel <= SIG_RTOL_F64 and cos >= 1 - COS_TOL_F64 and rank == l, (env, rel, cos, rank)


def test_paired_step_is_three_launches_and_matches_oracle():
    """The paired step (pair.cuh): k_gemv_n (w finalised in its tail),
    k_gemv_t2 on w, ONE k_cgs2_pair -- 3 launches per GK step -- and the
    bidiagonalization still meets the parity bar against the oracle."""
    from paper_2104_10785_b200 import _lib

    # 48 MB: not the resident kernel; rank 60, no breakdown within 40 steps
    A = synth.low_rank_synth(4000, 1500, 60, seed=12)
    op = K.DeviceMatrix.from_host(A)
    ctx = _lib.get_context()
    counts = {}
    for k in (20, 40):
        n0 = ctx.launch_count()
        K.bidiagonalize(op, K.BidiagConfig(k_max=k, seed=12))
        counts[k] = ctx.launch_count() - n0
    assert (counts[40] - counts[20]) == 3 * 20, counts
    ps = K.fsvd(op, k=80, r=20, cfg=K.BidiagConfig(k_max=80, seed=12))
    ref = O.fsvd_oracle(A, 80, 20, seed=12)
    assert np.max(np.abs(ps.sigma - ref.sigma) / ref.sigma) <= SIG_RTOL_F64
    cos = min(np.min(np.abs(np.einsum("ij,ij->j", ps.U, ref.U))),
              np.min(np.abs(np.einsum("ij,ij->j", ps.V, ref.V))))
    assert cos >= 1 - COS_TOL_F64
