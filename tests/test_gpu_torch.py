"""CUDA torch tensors as inputs (device-to-device, no host round trip):
row-major, transposed / strided views, f32 and non-float dtypes."""

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
from tests.parity import COS_TOL_F64, SIG_RTOL_F64, col_cos, sig_relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_cuda_tensors_all_layouts():
    A = synth.low_rank_synth(900, 600, 30, seed=3)
    ref = O.fsvd_oracle(A, 40, 10, seed=1)
    cfg = K.BidiagConfig(k_max=40, seed=1)
    base = torch.from_numpy(A).cuda()
    views = {"rowmajor": base,
             "transposed": torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t(),
             "strided": torch.from_numpy(np.repeat(A, 2, axis=1)).cuda()[:, ::2]}
    for name, t in views.items():
        assert torch.equal(t.cpu(), torch.from_numpy(A)), name
        ps = K.fsvd(t, k=40, r=10, cfg=cfg)
        assert sig_relerr(ps.sigma, ref.sigma) <= SIG_RTOL_F64, name
        assert np.min(col_cos(ps.U, ref.U)) >= 1 - COS_TOL_F64, name
    assert K.estimate_rank(base).rank == 30
    st = K.bidiagonalize(base, cfg)
    g = O.gk_oracle(A, 40, seed=1)
    assert st.terminated_early and abs(st.k_prime - g.k_prime) <= 2


def test_cuda_tensor_dtypes():
    A = synth.low_rank_synth(500, 300, 12, seed=4)
    t32 = torch.from_numpy(A.astype(np.float32)).cuda()
    op = K.as_operator(t32)
    assert op.dtype == np.float32 and np.array_equal(op.to_dense(), A.astype(np.float32))
    Ai = np.round(A * 10).astype(np.int32)
    opi = K.as_operator(torch.from_numpy(Ai).cuda())
    assert opi.dtype == np.float64 and np.array_equal(opi.to_dense(), Ai.astype(np.float64))
    with pytest.raises(K.ShapeMismatchError):
        K.as_operator(torch.zeros(5, device="cuda"))
