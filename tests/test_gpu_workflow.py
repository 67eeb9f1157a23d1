"""A user's workflow end to end through the public surfaces, in a
subprocess like a user would run it: the CLI writes a device-generated
snapshot, the CLI ranks it, Python streams it into HBM and runs fsvd,
the restarted mode and estimate_rank on the resident matrix."""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2104_10785_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_cli_gen_rank_then_python(tmp_path):
    snap = tmp_path / "a.klrm"
    res = _cli("gen", "--size", "6000x1500", "--kind", "harmonic", "--rank-true", "40",
               "--s0", "100", "--noise", "0", "--seed", "9", "--max-elems", "1e8",
               "--out", str(snap))
    assert res.returncode == 0, res.stderr[-2000:]
    res = _cli("rank", "--input", str(snap), "--eps", "1e-6", "--mode", "relative",
               "--repeats", "1", "--no-with-oracle", "--format", "json")
    assert res.returncode == 0, res.stderr[-2000:]
    doc = json.loads(res.stdout)
    assert doc["records"][0]["rank"] == 40 and doc["config"]["command"] == "rank"

    op = K.read_matrix_device(snap)
    A = K.read_matrix(snap)
    ps = K.fsvd(op, k=60, r=10, cfg=K.BidiagConfig(k_max=60, seed=2))
    ref = O.fsvd_oracle(A, 60, 10, seed=2)
    assert np.max(np.abs(ps.sigma - ref.sigma) / ref.sigma) <= 1e-10
    psr, info = K.fsvd_restarted(op, 10, k=24, tol=1e-11)
    exact = 100.0 / np.arange(1, 11)
    assert info.converged and np.max(np.abs(psr.sigma - exact) / exact) <= 1e-9
    assert K.estimate_rank(op, eps=1e-6, mode="relative").rank == 40
