"""Host-side logic of the drop-in API (CPU only): configuration validation,
the closed-form Gram tridiagonal, strict threshold counting, row sharding.
Cases restate the reference's unit tests (test_bidiag.py, test_fsvd.py,
test_rank.py)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2104_10785_b200 import (BidiagConfig, BidiagState, ConfigError, NumericalError,
                                   SymTridiag, bidiagonal_matrix, count_above, estimate_rank,
                                   fsvd, gram_tridiag, row_partition, substream, with_k_max)
from paper_2104_10785_b200.bidiag import bidiagonalize


def make_state(alphas, betas):
    a = np.asarray(alphas, dtype=np.float64)
    b = np.asarray(betas, dtype=np.float64)
    k = a.shape[0]
    return BidiagState(alphas=a, betas=b, Q=np.zeros((k + 1, k + 1)), P=np.zeros((k, k)),
                       k_prime=k, terminated_early=False)


def test_config_validation():
    with pytest.raises(ConfigError):
        BidiagConfig(k_max=0)
    with pytest.raises(ConfigError):
        BidiagConfig(k_max=2, eps=0.0)
    with pytest.raises(ConfigError):
        BidiagConfig(k_max=2, reorth_passes=3)
    with pytest.raises(ConfigError):
        BidiagConfig(k_max=2, start_std=0.0)
    c = BidiagConfig(k_max=3, seed=5)
    assert with_k_max(c, 3) is c and with_k_max(c, 7).k_max == 7


def test_entry_points_validate_before_touching_the_device():
    with pytest.raises(ConfigError):
        fsvd(np.eye(4), k=4, r=0)
    with pytest.raises(ConfigError):
        fsvd(np.eye(4), k=2, r=3)
    with pytest.raises(ConfigError):
        fsvd(np.eye(4), k=5, r=1)
    with pytest.raises(ConfigError):
        estimate_rank(np.eye(3), mode="fuzzy")
    with pytest.raises(ConfigError):
        estimate_rank(np.eye(3), eps=-1.0)
    with pytest.raises(ConfigError):
        bidiagonalize(np.eye(4), BidiagConfig(k_max=5))


def test_gram_hand_cases():
    tri = gram_tridiag(make_state([2.0, 3.0], [5.0, 4.0, 1.0]))
    assert np.array_equal(tri.diag, [20.0, 10.0])
    assert np.array_equal(tri.offdiag, [12.0])
    tri = gram_tridiag(make_state([3.0], [7.0, 0.5]))
    assert np.array_equal(tri.diag, [9.25]) and tri.offdiag.shape == (0,)


def test_gram_matches_explicit_product():
    rng = np.random.default_rng(3)
    a, b = rng.random(12) + 0.1, rng.random(13) + 0.1
    st_ = make_state(a, b)
    B = bidiagonal_matrix(st_)
    T = gram_tridiag(st_).to_dense()
    assert np.allclose(T, B.T @ B, rtol=1e-13, atol=1e-13)


def test_gram_degenerate_and_shape_errors():
    st_ = BidiagState(np.zeros(0), np.ones(1), np.zeros((3, 1)), np.zeros((2, 0)), 0, True, True)
    with pytest.raises(NumericalError):
        gram_tridiag(st_)
    with pytest.raises(ConfigError):
        SymTridiag(diag=np.ones(3), offdiag=np.ones(3))


def test_count_above_kats():
    theta = np.array([1.0, 1e-8, 1e-24])
    assert count_above(theta, 1e-8, "absolute") == (1, 1e-8)
    assert count_above(theta, 1e-9, "absolute")[0] == 2
    assert count_above(np.array([1.0, 0.5]), 0.5, "absolute")[0] == 1
    n, thr = count_above(np.array([4.0, 1e-6]), 1e-2, "relative")
    assert thr == 1e-4 * 4.0 and n == 1
    assert count_above(np.array([4.0, 1e-6]), 1e-4, "relative")[0] == 2
    assert count_above(np.zeros(0), 1e-8, "absolute") == (0, 1e-8)
    assert count_above(np.zeros(0), 1e-8, "relative") == (0, 0.0)
    with pytest.raises(ConfigError):
        count_above(np.ones(2), 1e-8, "fuzzy")
    with pytest.raises(ConfigError):
        count_above(np.ones(2), 0.0)


@settings(max_examples=30, deadline=None)
@given(st.lists(st.floats(1e-20, 1e10), min_size=1, max_size=30),
       st.floats(1e-20, 1e5), st.floats(1.0, 1e6))
def test_count_monotone_in_eps(vals, eps, factor):
    theta = np.sort(np.asarray(vals))[::-1]
    assert count_above(theta, eps * factor)[0] <= count_above(theta, eps)[0]


@settings(max_examples=50, deadline=None)
@given(st.integers(0, 10**6), st.integers(1, 64))
def test_row_partition_covers_rows_once(m, world):
    rows = []
    prev_end = 0
    for r in range(world):
        r0, ml = row_partition(m, world, r)
        assert r0 == prev_end and ml >= 0
        assert ml in (m // world, m // world + 1)
        prev_end = r0 + ml
        rows.append(ml)
    assert prev_end == m and sum(rows) == m


def test_substream_matches_reference_contract():
    a = substream(4, 1).standard_normal(8)
    assert np.array_equal(a, substream(4, 1).standard_normal(8))
    assert not np.array_equal(a, substream(4, 2).standard_normal(8))
    with pytest.raises(ConfigError):
        substream(None, 1)


def test_factored_operator_shape_errors_before_device_work():
    import paper_2104_10785_b200 as K
    with pytest.raises(K.ShapeMismatchError):
        K.FactoredOperator(np.ones((5, 3)), np.ones((2, 2)), np.ones((4, 2)))
    with pytest.raises(K.ShapeMismatchError):
        K.FactoredOperator(np.ones((5, 2)), np.ones((2, 3)), np.ones((4, 2)))
    with pytest.raises(K.ShapeMismatchError):
        K.FactoredOperator(np.ones(5), np.ones((1, 1)), np.ones((4, 1)))
