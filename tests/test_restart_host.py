"""Host logic of the restarted mode (paper_2104_10785_b200/restart.py): the
projected matrix T for every cycle / breakdown shape, and config errors
raised before any device work."""

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import _lib
from paper_2104_10785_b200.restart import _projected

A_ = np.array([3.0, 2.5, 2.0, 1.5, 1.0, 0.5])
B_ = np.array([9.0, 0.9, 0.8, 0.7, 0.6, 0.4, 0.3])  # betas[0] = beta_1 (unused)


def test_first_cycle_is_upper_bidiagonal():
    T, kq, kp = _projected(A_, B_, 6, 0)
    assert (kq, kp) == (6, 6)
    assert np.array_equal(np.diag(T), A_)
    assert np.array_equal(np.diag(T, 1), B_[1:6])
    assert np.count_nonzero(np.tril(T, -1)) == 0 and np.count_nonzero(np.triu(T, 2)) == 0


def test_beta_breakdown_truncates():
    T, kq, kp = _projected(A_, B_, 4, _lib.RUN_EARLY | _lib.RUN_BETA_BREAK)
    assert T.shape == (4, 4) and (kq, kp) == (4, 4)
    assert np.array_equal(np.diag(T), A_[:4]) and np.array_equal(np.diag(T, 1), B_[1:4])


def test_alpha_breakdown_adds_the_zero_column():
    T, kq, kp = _projected(A_, B_, 4, _lib.RUN_EARLY | _lib.RUN_ALPHA_BREAK)
    assert T.shape == (5, 5) and (kq, kp) == (5, 4)
    assert T[3, 4] == B_[4] and T[4, 4] == 0.0
    assert np.array_equal(np.diag(T)[:4], A_[:4])


def test_after_restart_spike_then_bidiagonal():
    s_l, rho = np.array([5.0, 4.0, 3.5]), np.array([0.1, -0.2, 0.05])
    a = np.zeros(7)
    b = np.zeros(8)
    a[3:] = [2.0, 1.8, 1.6, 1.4]  # alpha_{l+1..k}
    b[4:] = [0.7, 0.6, 0.5, 0.45]  # beta_{l+2..k+1}
    T, kq, kp = _projected(a, b, 7, 0, head=(s_l, rho))
    assert T.shape == (7, 7)
    assert np.array_equal(T[:3, :3], np.diag(s_l))
    assert np.array_equal(T[:3, 3], rho) and T[3, 3] == 2.0
    assert np.array_equal(np.diag(T)[3:], a[3:])
    assert np.array_equal(np.diag(T, 1)[3:], b[4:7])
    assert T[2, 3] == rho[2] and np.count_nonzero(np.tril(T, -1)) == 0


def test_alpha_breakdown_right_after_restart():
    s_l, rho = np.array([5.0, 4.0]), np.array([0.1, -0.2])
    T, kq, kp = _projected(np.zeros(6), np.zeros(7), 2, _lib.RUN_EARLY | _lib.RUN_ALPHA_BREAK,
                           head=(s_l, rho))
    assert T.shape == (3, 3) and (kq, kp) == (3, 2)
    assert np.array_equal(T[:2, 2], rho) and T[2, 2] == 0.0


@pytest.mark.parametrize("kw", [dict(r=0), dict(r=5, k=4), dict(r=5, k=10, keep=4),
                                dict(r=5, k=10, keep=10), dict(r=5, k=10, tol=-1.0)])
def test_config_errors_before_device_work(kw):
    with pytest.raises(K.ConfigError):
        K.fsvd_restarted(np.ones((40, 30)), **kw)
