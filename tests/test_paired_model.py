"""The paired GK step's arithmetic (DESIGN.md 3-pair, csrc/pair.cuh) against
the oracle on CPU: the reformulation -- A^T applied to the finalised but not
yet orthogonalised w, alpha = ||y'|| / beta -- meets the same parity
predicates as the device path (tests/parity.py), on low-rank, clustered,
rank-deficient-with-noise and f32-stored inputs.  No GPU involved."""

import numpy as np
import pytest

from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
from tests.paired_model import paired_gk
from tests.parity import assert_gk_match, ortho_dev


def _inputs():
    yield "low rank 400x300 r40", synth.low_rank_synth(400, 300, 40, seed=3), 60
    yield "gaussian 300x200", synth.gaussian_matrix(300, 200, seed=4), 80
    A = synth.config2_matrix(seed=1, m=2000, n=500, r=37)  # X Y^T + 1e-10 noise: past-rank steps
    yield "config-2 shape 2000x500 r37", A, 60
    yield "f32 entries", synth.low_rank_synth(500, 250, 30, seed=5).astype(np.float32).astype(np.float64), 50
    yield "config-1 matrix", synth.config1_matrix(seed=0), 30


@pytest.mark.parametrize("name,A,k", list(_inputs()), ids=lambda x: x if isinstance(x, str) else "")
def test_paired_step_matches_oracle(name, A, k):
    st = paired_gk(A, k, seed=7)
    ref = O.gk_oracle(A, k, seed=7)
    assert_gk_match(st["alphas"], st["betas"], st["k_prime"], ref.alphas, ref.betas,
                    ref.k_prime, what=name)
    # (after a breakdown the model leaves the terminal column out: Q[:, :k'])
    kq = st["k_prime"] + (1 if st["k_prime"] == k else 0)
    assert ortho_dev(st["Q"][:, :kq]) < 1e-10 and ortho_dev(st["P"]) < 1e-10, name
    # the GK relation A P = Q B holds for the paired recurrence too
    kp = st["k_prime"]
    if kp and kp == k:
        B = np.zeros((kp + 1, kp))
        B[np.arange(kp), np.arange(kp)] = st["alphas"]
        B[np.arange(1, kp + 1), np.arange(kp)] = st["betas"][1:]
        res = np.linalg.norm(A @ st["P"] - st["Q"] @ B) / np.linalg.norm(A)
        assert res < 1e-10, (name, res)
