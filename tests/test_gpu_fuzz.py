"""Seeded sweep over shapes, ranks, Krylov sizes and storage types against
the oracle: exercises every path-selection rule (resident whole-loop kernel,
tile-resident / global cooperative CGS, multi-kernel CGS, small-m U = A V,
single-CTA U filter) on shapes the hand-picked tests do not hit."""

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
from tests.parity import COS_TOL_F64, SIG_RTOL_F64, col_cos, gram_eigs

pytestmark = pytest.mark.gpu

NOISE_FLOOR = 1e-14  # x sigma_1: the eps ||A|| scale of post-rank Ritz values


def _cases(n_cases=36, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        m = int(rng.choice([rng.integers(1, 64), rng.integers(64, 700), rng.integers(700, 4000)]))
        n = int(rng.choice([rng.integers(1, 64), rng.integers(64, 700), rng.integers(700, 3000)]))
        kmax = min(m, n)
        l = int(rng.integers(1, kmax + 1))
        k = int(rng.integers(1, min(kmax, 160) + 1))
        r = int(rng.integers(1, k + 1))
        f32 = bool(rng.random() < 0.25)
        out.append((i, m, n, l, k, r, f32))
    return out


def _blocked(A):
    """The same matrix behind a row-block operator: the oracle with another
    summation order, to measure how rounding-sensitive each quantity is."""
    m, n = A.shape
    return O.BlockOp(m, n, lambda i0, i1: A[i0:i1], block=37)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c[1]}x{c[2]}-l{c[3]}-k{c[4]}"
                         + ("-f32" if c[6] else ""))
def test_fuzz_vs_oracle(case):
    """Ritz values of an UNconverged Krylov space on a clustered spectrum
    (products of Gaussians) move under a mere change of summation order --
    the oracle against itself with row-blocked products differs by up to
    ~1e-6 theta_1 on some of these shapes.  So every quantity is held to
    1e-10 OR to 10x the oracle's own summation-order spread, whichever is
    larger; the leading alphas/betas, the converged values, k' and the rank
    are held to the fixed tolerances.  Singular values below the numerical
    rank (post-rank Ritz values of a rank-l matrix, ~1e-9 sigma_1) are
    rounding artefacts of size eps ||A||: they additionally get the absolute
    floor NOISE_FLOOR * sigma_1 (Weyl: any backward-stable computation moves
    them by O(eps ||A||)); above ~1e-4 sigma_1 the floor is below 1e-10
    relative and changes nothing."""
    i, m, n, l, k, r, f32 = case
    A = synth.low_rank_synth(m, n, l, seed=1000 + i)
    if f32:
        A = A.astype(np.float32)
    A64 = A.astype(np.float64)
    cfg = K.BidiagConfig(k_max=k, seed=i)
    st = K.bidiagonalize(A, cfg)
    ref = O.gk_oracle(A64, k, seed=i)
    ref2 = O.gk_oracle(_blocked(A64), k, seed=i)
    assert st.degenerate == ref.degenerate
    assert abs(st.k_prime - ref.k_prime) <= 2, case
    h = min(8, len(st.alphas), len(ref.alphas))
    if h:
        assert np.max(np.abs(st.alphas[:h] - ref.alphas[:h])) <= \
            SIG_RTOL_F64 * np.max(np.abs(ref.alphas)), case
    th, rth, rth2 = (gram_eigs(x.alphas, x.betas) for x in (st, ref, ref2))
    nt = min(len(th), len(rth), len(rth2))
    if nt:
        tol = np.maximum(SIG_RTOL_F64 * rth[0], 10 * np.abs(rth[:nt] - rth2[:nt]))
        assert np.all(np.abs(th[:nt] - rth[:nt]) <= tol), case
    ps = K.fsvd(A, k=k, r=r, cfg=cfg)
    fr = O.fsvd_oracle(A64, k, r, seed=i)
    fr2 = O.fsvd_oracle(_blocked(A64), k, r, seed=i)
    nt = min(ps.sigma.size, fr.sigma.size, fr2.sigma.size)
    assert abs(ps.sigma.size - fr.sigma.size) <= max(0, fr.sigma.size - nt) + 0, case
    if nt:
        spread = np.abs(fr.sigma[:nt] - fr2.sigma[:nt])
        tol = np.maximum(np.maximum(SIG_RTOL_F64 * fr.sigma[:nt], 10 * spread),
                         NOISE_FLOOR * fr.sigma[0])
        assert np.all(np.abs(ps.sigma[:nt] - fr.sigma[:nt]) <= tol), case
        stable = spread <= 1e-12 * fr.sigma[:nt]
        if stable.any():
            cos = col_cos(ps.V[:, :nt][:, stable], fr.V[:, :nt][:, stable])
            assert np.min(cos) >= 1 - COS_TOL_F64, case
    assert K.estimate_rank(A).rank == O.rank_oracle(A64).rank, case


def test_fuzz_streaming_paths():
    """The same sweep with the whole-loop resident kernel disabled
    (KSVD_RESIDENT=0): every shape then runs the streaming kernels -- the
    paired step (k_cgs2_pair) where its tiles fit, else the serialised one."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          f"{Path(__file__).resolve()}::test_fuzz_vs_oracle"],
                         cwd=root, env={**os.environ, "KSVD_RESIDENT": "0"},
                         capture_output=True, text=True, timeout=1200)
    assert res.returncode == 0, res.stdout[-3000:]
