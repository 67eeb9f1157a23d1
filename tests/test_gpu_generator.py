"""On-device generator of BASELINE.json configs 3-5 (include/ksvd_gen.h):
rows are bit-identical to the host regeneration used by the oracle, the
factors are orthonormal, and fsvd / estimate_rank on generated matrices
match the CPU oracle run on the regenerated rows."""

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from oracle.generated import GeneratedRows, host_normal
from paper_2104_10785_b200 import synth
from tests.parity import (COS_TOL_F64, SIG_RTOL_F32, SIG_RTOL_F64, col_cos, ortho_dev,
                          sig_relerr)

pytestmark = pytest.mark.gpu

SMALL = {
    3: synth.BASELINE_SPECS[3].scaled(6000, 1500),
    4: synth.BASELINE_SPECS[4].scaled(8000, 2000),
    5: synth.BASELINE_SPECS[5].scaled(6000, 1200),
}


def regen(op, spec):
    ps, q = op.gen_factors()
    return GeneratedRows(ps, q, spec.noise, spec.seed, spec.dtype == "f32", row0=op.row0)


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_rows_bit_identical_to_host(cfg):
    spec = SMALL[cfg]
    op = synth.generate(spec)
    rows = regen(op, spec)
    A_dev = op.to_dense().astype(np.float64)
    for i0, i1 in [(0, 7), (1234, 1300), (spec.m - 5, spec.m)]:
        assert np.array_equal(A_dev[i0:i1], rows(i0, i1)), (cfg, i0)
    # factors: P and Q orthonormal, Ps = P diag(s)
    ps, q = op.gen_factors()
    assert ortho_dev(q) < 1e-13
    s = np.linalg.norm(ps, axis=0)
    assert np.all(np.diff(s) <= 1e-12 * s[0])  # descending spectrum
    assert ortho_dev(ps / s) < 1e-13


def test_noise_stream_is_gaussian():
    x = np.array([host_normal(7, 1, i) for i in range(50000)])
    assert abs(x.mean()) < 0.02 and abs(x.std() - 1) < 0.02


@pytest.mark.parametrize("cfg", [3, 4])
def test_fsvd_generated_vs_oracle(cfg):
    spec = SMALL[cfg]
    call = synth.BASELINE_CALLS[cfg]
    op = synth.generate(spec)
    A = regen(op, spec)(0, spec.m)  # the same entries, on the host
    k, r = min(call["k"], spec.n), min(call["r"], spec.n)
    ours = K.fsvd(op, k=k, r=r, cfg=K.BidiagConfig(k_max=k, seed=call["seed"]))
    ref = O.fsvd_oracle(A, k, r, seed=call["seed"])
    tol = SIG_RTOL_F32 if spec.dtype == "f32" else SIG_RTOL_F64
    assert sig_relerr(ours.sigma, ref.sigma) <= tol
    # f64 accumulation makes the f32-stored case fp64-accurate as well
    assert sig_relerr(ours.sigma, ref.sigma) <= SIG_RTOL_F64
    assert np.min(col_cos(ours.V, ref.V)) >= 1 - COS_TOL_F64
    assert np.min(col_cos(ours.U, ref.U)) >= 1 - COS_TOL_F64
    res = np.linalg.norm(A @ ours.V - ours.U * ours.sigma, axis=0)
    assert np.max(res) <= 1e-4 * ours.sigma[0]


def test_rank_generated_vs_oracle():
    spec = SMALL[5]
    call = synth.BASELINE_CALLS[5]
    op = synth.generate(spec)
    A = regen(op, spec)(0, spec.m)
    ours = K.estimate_rank(op, eps=call["eps"], mode=call["mode"],
                           cfg=K.BidiagConfig(k_max=1, seed=call["seed"]))
    ref = O.rank_oracle(A, eps=call["eps"], mode=call["mode"], seed=call["seed"])
    assert ours.rank == ref.rank == spec.rank
