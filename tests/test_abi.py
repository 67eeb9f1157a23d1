"""The C-ABI library: loads, exports every symbol include/ksvd.h declares,
and its host-side spectral stage matches the reference (CPU only; no
compute call touches a GPU here)."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2104_10785_b200 import _lib, symtridiag_eig, SymTridiag
from paper_2104_10785_b200.build import LIB, needs_build
from tests.parity import col_cos

HEADER = Path(__file__).resolve().parent.parent / "include" / "ksvd.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ksvd_[a-z0-9_]+)\s*\(", text)))


def test_library_built_and_loads():
    assert LIB.exists(), "run python -m paper_2104_10785_b200.build"
    assert not needs_build(), "libksvd.so is older than its sources"
    lib = _lib.load_library()
    assert lib.ksvd_version() == 1


def test_exports_every_declared_symbol():
    lib = _lib.load_library()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    # and the ctypes table binds exactly the header's surface
    assert sorted(_lib.SIGNATURES) == syms


def test_sm100a_code_in_library():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout[:500]


@pytest.mark.parametrize("n", [1, 2, 3, 5, 13, 50, 120])
def test_native_eig_matches_reference_kat(golden, n):
    d, e = golden[f"eig/{n}/d"], golden[f"eig/{n}/e"]
    theta, G = symtridiag_eig(SymTridiag(d, e))
    tref, Gref = golden[f"eig/{n}/theta"], golden[f"eig/{n}/G"]
    scale = max(np.max(np.abs(tref)), 1.0)
    assert np.max(np.abs(theta - tref)) <= 1e-12 * scale
    assert np.min(col_cos(G, Gref)) >= 1 - 1e-10
    assert np.max(np.abs(G.T @ G - np.eye(n))) < 1e-12


def test_native_eig_no_vectors_and_errors():
    theta, G = symtridiag_eig(SymTridiag(np.array([1.0, 2.0]), np.array([0.5])), vectors=False)
    assert G is None and theta.shape == (2,)
    from paper_2104_10785_b200 import ConfigError

    with pytest.raises(ConfigError):
        symtridiag_eig(SymTridiag(np.zeros(0), np.zeros(0)))


def test_no_cpu_fallback_without_gpu():
    """On a host without a GPU every compute entry point fails loudly."""
    import ctypes as C

    lib = _lib.load_library()
    n = C.c_int(0)
    rc = lib.ksvd_device_count(C.byref(n))
    if rc == 0 and n.value > 0:
        pytest.skip("a GPU is visible")
    from paper_2104_10785_b200 import fsvd

    _lib.set_context(None)
    with pytest.raises(RuntimeError):
        fsvd(np.eye(4), k=2, r=1)


def test_bidiag_sv2_relative_accuracy():
    """Rank estimation's tiny bidiagonal SVD (eig.cpp ksvd_bidiag_sv2): the
    tail below 1e-6 theta_1 is accurate to a few ulps of each value (a QL on
    B^T B only resolves it to eps*||T||), the head to eps*theta_1 like the
    reference's QL (checked against 50-digit arithmetic)."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 50
    rng = np.random.default_rng(11)
    for k, graded in [(1, False), (7, False), (40, False), (25, True)]:
        a = rng.random(k) + 0.1
        b = rng.random(k + 1) + 0.1
        if graded:
            a = a * 10.0 ** (-0.9 * np.arange(k))
            b[1:] = b[1:] * 10.0 ** (-0.9 * np.arange(k))
        B = np.zeros((k + 1, k))
        B[np.arange(k), np.arange(k)] = a
        B[np.arange(1, k + 1), np.arange(k)] = b[1:]
        ref = sorted((float(x) ** 2 for x in mpmath.svd_r(mpmath.matrix(B.tolist()),
                                                            compute_uv=False)), reverse=True)
        got = _lib.bidiag_sv2(a, b)
        ref = np.array(ref)
        tail = ref < 1e-6 * ref[0]  # bisection: relative accuracy
        assert np.all(np.abs(got - ref)[tail] / ref[tail] < 1e-14), (k, graded)
        # head: QL on B^T B, like the reference (absolute eps*theta_1)
        assert np.max(np.abs(got - ref)[~tail]) < 1e-13 * ref[0], (k, graded)


def test_dense_svd_native_matches_numpy():
    """ksvd_dense_svd (host Jacobi, restarted mode's projected matrix)."""
    from paper_2104_10785_b200.restart import dense_svd
    rng = np.random.default_rng(3)
    for k in (1, 2, 7, 40, 120):
        T = np.triu(rng.standard_normal((k, k)))
        T[: k // 3, : k // 3] = np.diag(np.sort(rng.uniform(1, 5, k // 3))[::-1])
        Uh, s, Vh = dense_svd(T)
        ref = np.linalg.svd(T, compute_uv=False)
        assert np.allclose(s, ref, rtol=1e-13, atol=1e-15 * ref[0])
        assert np.allclose(Uh * s @ Vh.T, T, atol=1e-13 * ref[0])
        assert np.allclose(Vh.T @ Vh, np.eye(k), atol=1e-13)
    # graded: tiny singular values to high relative accuracy
    T = np.diag(10.0 ** -np.arange(0, 16, 2.0)) @ np.triu(np.ones((8, 8)) * 0.1 + np.eye(8))
    s = dense_svd(T)[1]
    assert np.all(s > 0) and s[-1] < 1e-13
