"""Full-size golden fixtures for BASELINE configs 3 and 5 (and 4 when run).

Two steps:

1. On the GPU box (196 GB host RAM, 16 cores), `tools/fullsize_oracle.py
   --config N` generates A in HBM, runs this package's entry point, downloads
   the SAME bits and runs the CPU oracle (oracle/krylov_oracle.py) on them;
   it writes gpurun_out/fullsize/cN.npz.
2. Here, where the reference imports:

       PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_golden.py

   keeps the oracle's outputs (subsampled rows of U and V) and adds the
   REFERENCE's own eigen-solve (krysvd.fsvd.symtridiag_eig on the Gram
   tridiagonal, rank.py:64) and count (rank.py:33-48) on the oracle's
   alphas/betas and on the GPU's -- the count the reference itself would
   report on each Krylov run.

Writes tests/golden/full_c3.npz, full_c5.npz (and full_c4.npz).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from krysvd.fsvd import SymTridiag, symtridiag_eig  # noqa: E402  (the reference)
from krysvd.rank import count_above  # noqa: E402

SRC = ROOT / "gpurun_out" / "fullsize"
VROWS = 2000  # rows of V kept (evenly spaced); U rows are already subsampled


def ref_count(alphas, betas, eps, mode):
    a = np.asarray(alphas, np.float64)
    b = np.asarray(betas, np.float64)
    theta = symtridiag_eig(SymTridiag(a * a + b[1:] ** 2, a[1:] * b[1:-1]), vectors=False)
    theta = theta[0] if isinstance(theta, tuple) else theta
    return count_above(theta, eps, mode)[0], theta


def fsvd_case(cfg: int):
    d = dict(np.load(SRC / f"c{cfg}.npz"))
    n = d["oracle_V"].shape[0]
    vrows = np.linspace(0, n - 1, min(VROWS, n)).astype(np.int64)
    out = {k: d[k] for k in ("oracle_sigma", "oracle_U_rows", "urows", "oracle_alphas",
                             "oracle_betas", "oracle_kprime", "oracle_theta")}
    out["oracle_V_rows"] = d["oracle_V"][vrows]
    out["vrows"] = vrows
    np.savez_compressed(HERE / f"full_c{cfg}.npz", **out)
    print(f"config {cfg}: k' {int(d['oracle_kprime'])}, sigma {d['oracle_sigma'][:3]}")


def rank_case(cfg: int, eps: float, mode: str):
    d = dict(np.load(SRC / f"c{cfg}.npz"))
    ro, th_o = ref_count(d["oracle_alphas"], d["oracle_betas"], eps, mode)
    rg, _ = ref_count(d["gpu_alphas"], d["gpu_betas"], eps, mode)
    out = {k: d[k] for k in ("oracle_alphas", "oracle_betas", "oracle_kprime", "oracle_rank",
                             "oracle_theta")}
    out.update(reference_ql_rank_on_oracle=ro, reference_ql_theta_on_oracle=th_o,
               reference_ql_rank_on_gpu=rg, gpu_alphas_at_generation=d["gpu_alphas"],
               gpu_betas_at_generation=d["gpu_betas"])
    np.savez_compressed(HERE / f"full_c{cfg}.npz", **out)
    print(f"config {cfg}: oracle QL rank {int(d['oracle_rank'])}, reference QL on oracle "
          f"alphas/betas {ro}, reference QL on GPU alphas/betas {rg}, k' "
          f"{int(d['oracle_kprime'])}")


if __name__ == "__main__":
    fsvd_case(3)
    rank_case(5, 1e-8, "relative")
    if (SRC / "c4.npz").exists():
        fsvd_case(4)
