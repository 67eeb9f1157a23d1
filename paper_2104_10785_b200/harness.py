"""Benchmark-harness operations behind the CLI (reference bench.py:1-283,
restricted to the GK path): method runs, error metrics and timing, with the
reference's record schema so GPU and oracle tables diff line by line.

Methods: "fsvd" runs this package's GPU path; "dense" is the reference's
LAPACK cross-check (bench.py:114-117, linops.py:288-300) and runs on the host
exactly as there -- it is a labelled comparison column, not a fallback for
the GPU path.  The randomized-SVD methods and the RSL trainer are outside
the hot-path scope and raise ConfigError.

Timing protocol (bench.py:1-7): one discarded warm-up, then `repeats` runs
on a monotonic clock; the median is the headline and the mean rides along.
An ndarray input is uploaded inside every timed call, as the reference
times its host arrays.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .bidiag import BidiagConfig
from .errors import ConfigError
from .fsvd import fsvd
from .linops import BENCH_MATRIX, BENCH_METHOD, PartialSvd, derive_seed
from .rank import count_above, estimate_rank
from .synth import low_rank_synth

SCHEMA_VERSION = 1
METHODS = ("fsvd", "rsvd-default", "rsvd-oversampled", "dense")  # reference set
GPU_METHODS = ("fsvd", "dense")
ERR_RES_CAP = 10 ** 8
ORACLE_CAP = 1024


@dataclass(frozen=True)
class BenchRecord:
    """One compare row; field order is the pinned CSV header."""

    method: str
    m: int
    n: int
    rank_true: int
    r_extracted: int
    k_used: int
    seconds: float
    seconds_mean: float
    err_res: float | None
    err_res_full: float | None
    err_rel: float
    rank_estimated: int | None
    seed: int


@dataclass(frozen=True)
class TripletQuality:
    method: str
    q: np.ndarray
    sigma_oracle: np.ndarray
    sigma_method: np.ndarray


def parse_size(text: str) -> tuple[int, int]:
    parts = text.lower().split("x")
    if len(parts) != 2:
        raise ConfigError(f"size must look like 1000x1000, got {text!r}")
    try:
        return int(parts[0]), int(parts[1])
    except ValueError as exc:
        raise ConfigError(f"size must look like 1000x1000, got {text!r}") from exc


def _host(A) -> np.ndarray:
    return A if isinstance(A, np.ndarray) else A.to_dense()


def err_rel(A, psvd: PartialSvd) -> float:
    """||A^T U - V Sigma||_F / ||Sigma||_F (bench.py:61-68)."""
    denom = float(np.linalg.norm(psvd.sigma))
    if denom == 0.0:
        return float("nan")
    R = _host(A).T @ psvd.U - psvd.V * psvd.sigma
    return float(np.linalg.norm(R)) / denom


def err_res(A, psvd: PartialSvd) -> float:
    """||A - U Sigma V^T||_F, materialized (bench.py:71-74)."""
    return float(np.linalg.norm(_host(A) - (psvd.U * psvd.sigma) @ psvd.V.T))


def dense_svd(A) -> PartialSvd:
    """All triplets via LAPACK, signs fixed like fix_signs (linops.py:271-282)."""
    A = _host(A)
    if min(A.shape) > ORACLE_CAP:
        raise ConfigError(f"dense oracle capped at min(m,n) <= {ORACLE_CAP}, got shape {A.shape}")
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    V = Vt.T
    if V.shape[1]:
        lead = V[np.argmax(np.abs(V), axis=0), np.arange(V.shape[1])]
        sgn = np.where(lead < 0, -1.0, 1.0)
        U, V = U * sgn, V * sgn
    return PartialSvd(U=U, sigma=s, V=V)


def triplet_quality(oracle: PartialSvd, method_psvd: PartialSvd, name: str) -> TripletQuality:
    """q_j = <u_j, u_j'> <v_j, v_j'> against the oracle (bench.py:79-85)."""
    r = min(oracle.rank, method_psvd.rank)
    qu = np.einsum("ij,ij->j", oracle.U[:, :r], method_psvd.U[:, :r])
    qv = np.einsum("ij,ij->j", oracle.V[:, :r], method_psvd.V[:, :r])
    return TripletQuality(name, qu * qv, oracle.sigma[:r].copy(), method_psvd.sigma[:r].copy())


def run_method(method: str, A, r: int, rank_true: int | None, seed: int,
               k: int | None = None, power_iters: int = 0,
               oversampling: int | None = None) -> dict:
    """One factorization (bench.py:86-133): psvd_r (r triplets), psvd_full
    (everything computed), k_used and the method's rank estimate."""
    m, n = A.shape
    if method not in METHODS:
        raise ConfigError(f"unknown method {method!r}, expected one of {METHODS}")
    if method not in GPU_METHODS:
        raise ConfigError(f"method {method!r} is outside this package's scope "
                          f"(supported: {', '.join(GPU_METHODS)})")
    if not 1 <= r <= min(m, n):
        raise ConfigError(f"r must be in [1, min(m,n)] = [1, {min(m, n)}], got {r}")
    if method == "dense":
        full = dense_svd(A)
        return {"psvd_r": full.top(r), "psvd_full": full, "k_used": min(m, n),
                "rank_estimated": None}
    kk = min(m, n) if k is None else k
    full, state, theta = fsvd(A, k=kk, r=kk, cfg=BidiagConfig(k_max=kk, seed=seed),
                              return_details=True)
    est = count_above(theta, 1e-8, "absolute")[0] if theta.size else 0
    return {"psvd_r": full.top(r), "psvd_full": full, "k_used": state.k_prime,
            "rank_estimated": est}


def timed(fn, repeats: int):
    """(last result, median seconds, mean seconds) after one warm-up."""
    fn()
    out, ts = None, []
    for _ in range(repeats):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return out, float(np.median(ts)), float(np.mean(ts))


def _check_cap(m: int, n: int, cap: float) -> None:
    if m * n > cap:
        raise ConfigError(f"size {m}x{n} exceeds the element cap {cap:g}")


def _dense_rank(A, eps: float, mode: str, repeats: int):
    def count():
        s = np.linalg.svd(_host(A), compute_uv=False)
        return count_above(s * s, eps, mode)[0]
    rank, med, _ = timed(count, repeats)
    return rank, med


def _rank_row(A, rank_true, eps, mode, cfg, repeats, seed, with_oracle) -> dict:
    m, n = A.shape
    rep, med, mean = timed(lambda: estimate_rank(A, eps=eps, mode=mode, cfg=cfg), repeats)
    row = {"m": m, "n": n, "rank_true": rank_true, "rank": rep.rank, "k_prime": rep.k_prime,
           "eps": eps, "mode": mode, "threshold": rep.threshold, "seconds": med,
           "seconds_mean": mean, "oracle_rank": None, "oracle_seconds": None, "seed": seed}
    if with_oracle and min(m, n) <= ORACLE_CAP:
        row["oracle_rank"], row["oracle_seconds"] = _dense_rank(A, eps, mode, repeats)
    return row


def cmd_rank(sizes, rank_true: int, eps: float = 1e-8, mode: str = "absolute",
             repeats: int = 3, seed: int = 0, with_oracle: bool = True,
             max_elems: float = 1e8) -> list[dict]:
    """Rank rows for synthetic low-rank matrices (bench.py:189-219)."""
    if repeats < 1:
        raise ConfigError(f"repeats must be >= 1, got {repeats}")
    rows = []
    for si, (m, n) in enumerate(sizes):
        _check_cap(m, n, max_elems)
        A = low_rank_synth(m, n, rank_true, seed=derive_seed(seed, BENCH_MATRIX, si))
        cfg = BidiagConfig(k_max=min(m, n), seed=derive_seed(seed, BENCH_METHOD, si))
        rows.append(_rank_row(A, rank_true, eps, mode, cfg, repeats, seed, with_oracle))
    return rows


def rank_report_for_matrix(A, eps: float = 1e-8, mode: str = "absolute", seed: int = 0,
                           repeats: int = 3, with_oracle: bool = True) -> dict:
    """Single-matrix rank row for file inputs (bench.py:222-243)."""
    cfg = BidiagConfig(k_max=min(A.shape), seed=seed)
    return _rank_row(A, None, eps, mode, cfg, max(repeats, 1), seed, with_oracle)


def cmd_svd(A, method: str, r: int, rank_true: int | None = None, k: int | None = None,
            repeats: int = 3, seed: int = 0, power_iters: int = 0,
            oversampling: int | None = None, max_elems: float = 1e8):
    """(per-index sigma rows, summary) for one method on one matrix
    (bench.py:246-266)."""
    m, n = A.shape
    res, med, mean = timed(lambda: run_method(method, A, r, rank_true, seed, k=k,
                                              power_iters=power_iters,
                                              oversampling=oversampling), max(repeats, 1))
    ps = res["psvd_r"]
    small = m * n <= min(ERR_RES_CAP, max_elems)
    summary = {"method": method, "m": m, "n": n, "r": r, "k_used": res["k_used"],
               "rank_estimated": res["rank_estimated"], "err_rel": err_rel(A, ps),
               "err_res": err_res(A, ps) if small else None,
               "err_res_full": err_res(A, res["psvd_full"]) if small else None,
               "truncated": ps.truncated, "seconds": med, "seconds_mean": mean, "seed": seed}
    return [{"index": i + 1, "sigma": float(s)} for i, s in enumerate(ps.sigma)], summary


def cmd_compare(sizes, rank_true: int, r: int, methods, repeats: int = 3, seed: int = 0,
                max_elems: float = 1e8, power_iters: int = 0,
                oversampling: int | None = None) -> list[BenchRecord]:
    """Methods x sizes table (bench.py:149-186)."""
    if repeats < 1:
        raise ConfigError(f"repeats must be >= 1, got {repeats}")
    out = []
    for si, (m, n) in enumerate(sizes):
        _check_cap(m, n, max_elems)
        A = low_rank_synth(m, n, rank_true, seed=derive_seed(seed, BENCH_MATRIX, si))
        for mi, method in enumerate(methods):
            mseed = derive_seed(seed, BENCH_METHOD, si, mi)
            res, med, mean = timed(lambda: run_method(method, A, r, rank_true, mseed,
                                                      power_iters=power_iters,
                                                      oversampling=oversampling), repeats)
            small = m * n <= ERR_RES_CAP
            out.append(BenchRecord(
                method=method, m=m, n=n, rank_true=rank_true, r_extracted=r,
                k_used=res["k_used"], seconds=med, seconds_mean=mean,
                err_res=err_res(A, res["psvd_r"]) if small else None,
                err_res_full=err_res(A, res["psvd_full"]) if small else None,
                err_rel=err_rel(A, res["psvd_r"]), rank_estimated=res["rank_estimated"],
                seed=seed))
    return out


def cmd_triplet_quality(m: int, n: int, rank_true: int, r: int, methods, seed: int = 0,
                        power_iters: int = 0,
                        oversampling: int | None = None) -> list[TripletQuality]:
    """Per-direction agreement with the dense oracle (bench.py:269-283)."""
    if min(m, n) > ORACLE_CAP:
        raise ConfigError(f"triplet quality needs the dense oracle; "
                          f"min(m,n) must be <= {ORACLE_CAP}, got {m}x{n}")
    A = low_rank_synth(m, n, rank_true, seed=derive_seed(seed, BENCH_MATRIX, 0))
    ref = dense_svd(A).top(r)
    out = []
    for mi, method in enumerate(methods):
        ps = run_method(method, A, r, rank_true, derive_seed(seed, BENCH_METHOD, 0, mi),
                        power_iters=power_iters, oversampling=oversampling)["psvd_r"]
        j = min(ref.rank, ps.rank)
        q = np.sum(ref.U[:, :j] * ps.U[:, :j], axis=0) * np.sum(ref.V[:, :j] * ps.V[:, :j], axis=0)
        out.append(TripletQuality(method, q, ref.sigma[:j].copy(), ps.sigma[:j].copy()))
    return out
