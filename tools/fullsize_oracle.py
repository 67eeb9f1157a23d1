#!/usr/bin/env python
"""Full-size parity run for BASELINE configs 3-5 on the GPU box (host RAM
196 GB): generate A in HBM, run this package's entry point on it, download
the SAME bits (ksvd_matrix_to_host) and run the CPU oracle on them
(oracle/krylov_oracle.py, numpy/OpenBLAS on every host core).  Writes
gpurun_out/fullsize/c<N>.npz; tests/golden/make_fullsize_golden.py turns
that into the committed fixture (adding the reference's own QL count).

    python tools/fullsize_oracle.py --config 5
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2104_10785_b200 as K  # noqa: E402
from oracle import krylov_oracle as O  # noqa: E402
from paper_2104_10785_b200 import _lib, synth  # noqa: E402
from paper_2104_10785_b200.fsvd import _gram, symtridiag_eig  # noqa: E402


class F32RowsOp:
    """A held in f32 (config 4: 160 GB), products in f64 on the up-cast
    entries through the oracle's C helper (the reference coerces A to f64,
    linops.py:82-86; 320 GB would not fit the host)."""

    def __init__(self, A32):
        from oracle.generated import lib

        self.A = A32
        self.shape = A32.shape
        self.lib = lib()

    def apply(self, x):
        import ctypes as C

        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.shape[0])
        pd = C.POINTER(C.c_double)
        self.lib.ksvd_host_gemv_f32(self.A.ctypes.data_as(C.c_void_p), self.shape[0],
                                    self.shape[1], x.ctypes.data_as(pd), y.ctypes.data_as(pd))
        return y

    def apply_t(self, y):
        import ctypes as C

        y = np.ascontiguousarray(y, dtype=np.float64)
        z = np.empty(self.shape[1])
        pd = C.POINTER(C.c_double)
        self.lib.ksvd_host_gemv_t_f32(self.A.ctypes.data_as(C.c_void_p), self.shape[0],
                                      self.shape[1], y.ctypes.data_as(pd), z.ctypes.data_as(pd))
        return z

    def apply_many(self, X):
        return np.column_stack([self.apply(X[:, j]) for j in range(X.shape[1])])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=[3, 4, 5])
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "fullsize"))
    ap.add_argument("--urows", type=int, default=2000, help="U rows kept (evenly spaced)")
    a = ap.parse_args()
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    spec = synth.BASELINE_SPECS[a.config]
    call = synth.BASELINE_CALLS[a.config]
    log = {"config": a.config, "m": spec.m, "n": spec.n, "host_threads": os.cpu_count()}
    res = {}

    t0 = time.perf_counter()
    op = synth.generate(spec)
    _lib.get_context().sync()
    log["generate_s"] = time.perf_counter() - t0

    # ---- this package on the device ----
    if call["kind"] == "rank":
        cfg = K.BidiagConfig(k_max=1, seed=call["seed"])
        t0 = time.perf_counter()
        rep = K.estimate_rank(op, eps=call["eps"], mode=call["mode"], cfg=cfg)
        log["gpu_s"] = time.perf_counter() - t0
        run = K.run_gk(op, K.with_k_max(cfg, min(spec.m, spec.n)))
        res.update(gpu_rank=rep.rank, gpu_kprime=rep.k_prime, gpu_theta=rep.eigenvalues,
                   gpu_alphas=run.alphas, gpu_betas=run.betas)
        run.free()
        # the reference's method (Gram tridiagonal + QL, rank.py:64) on the GPU alphas/betas
        th_ql, _ = symtridiag_eig(_gram(res["gpu_alphas"], res["gpu_betas"]), vectors=False)
        res["gpu_theta_ql"] = th_ql
        res["gpu_rank_ql"] = K.count_above(th_ql, call["eps"], call["mode"])[0]
    else:
        cfg = K.BidiagConfig(k_max=call["k"], eps=call["eps"], seed=call["seed"])
        t0 = time.perf_counter()
        ps, st, theta = K.fsvd(op, k=call["k"], r=call["r"], cfg=cfg, return_details=True)
        log["gpu_s"] = time.perf_counter() - t0
        rows = np.linspace(0, spec.m - 1, a.urows).astype(np.int64)
        res.update(gpu_sigma=ps.sigma, gpu_V=ps.V, gpu_U_rows=ps.U[rows], urows=rows,
                   gpu_alphas=st.alphas, gpu_betas=st.betas, gpu_kprime=st.k_prime,
                   gpu_theta=theta)
        del ps, st
    print(json.dumps(log), flush=True)

    # ---- the same bits on the host ----
    t0 = time.perf_counter()
    A = op.to_dense()
    log["download_s"] = time.perf_counter() - t0
    op.free()
    _lib.get_context().release_pool()
    Aop = F32RowsOp(A) if A.dtype == np.float32 else A

    t0 = time.perf_counter()
    if call["kind"] == "rank":
        ro = O.rank_oracle(Aop, eps=call["eps"], mode=call["mode"], seed=call["seed"])
        log["oracle_s"] = time.perf_counter() - t0
        res.update(oracle_rank=ro.rank, oracle_kprime=ro.k_prime, oracle_theta=ro.eigenvalues,
                   oracle_alphas=ro.gk.alphas, oracle_betas=ro.gk.betas)
    else:
        fo = O.fsvd_oracle(Aop, call["k"], call["r"], eps=call["eps"], seed=call["seed"])
        log["oracle_s"] = time.perf_counter() - t0
        res.update(oracle_sigma=fo.sigma, oracle_V=fo.V, oracle_U_rows=fo.U[res["urows"]],
                   oracle_alphas=fo.gk.alphas, oracle_betas=fo.gk.betas,
                   oracle_kprime=fo.gk.k_prime, oracle_theta=fo.theta)
    log["host_threads_blas"] = _blas_threads()
    np.savez_compressed(out / f"c{a.config}.npz", **{k: np.asarray(v) for k, v in res.items()})
    (out / f"c{a.config}.json").write_text(json.dumps(log, indent=1))
    print(json.dumps(log), flush=True)
    summary = {k: (int(v) if np.ndim(v) == 0 else None) for k, v in res.items()}
    print(json.dumps({k: v for k, v in summary.items() if v is not None}), flush=True)


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info()), default=None)
    except Exception:  # noqa: BLE001
        return None


if __name__ == "__main__":
    main()
