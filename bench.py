#!/usr/bin/env python
"""Benchmark of the B200 GK bidiagonalization path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One bench "step" is one call of the reference entry point on configuration
C of BASELINE.json.  Default C = 4: `fsvd(A, k=96, r=32)` of the
1,000,000 x 40,000 f32 matrix (160 GB) -- the largest configuration that
fits one B200, the one `north_star` states its roofline target for.
Configs 1-2 are built on the host (numpy); 3-5 are generated in HBM
(include/ksvd_gen.h).  Metric: GK steps/s = GK iterations (k') per call /
time per call; the line also carries the time to result, the effective HBM
bandwidth 2 m n bytes k' / time, the roofline of the A-streaming kernels,
the CPU baseline and the end-to-end number through the public API.

  --gpus N : without torchrun, bench.py launches N ranks itself (one process
             per GPU, RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* set, N = 1
             included) and exits non-zero if fewer than N GPUs are visible.
             Under torchrun it is one of the ranks.  A is row-sharded over
             the ranks (strong scaling: the matrix is fixed).
  value    : device-resident A, CUDA events on the library stream around
             exactly K calls, barrier + sync on both sides, max over ranks.
             A is larger than L2 (126 MB) for every config but config 1
             (16 MB, L2-resident: latency-bound by construction).
  e2e      : the public call on a plain (pageable) numpy copy of this rank's
             rows: upload (libksvd stages it through pinned chunks) + the run
             + the read-back of the result, every step; for the generated
             configs the host copy is downloaded once after the device
             measurements and the resident matrix is freed first.  The
             one-off ingestion (generator / upload rate) is reported in
             `ingest`.
  roofline : per-launch CUDA-event durations of gemv_n / gemv_t measured in
             a profiled repeat of the same calls; algorithmic bytes per
             launch = m_local * n * sizeof(A).
  --impl reference : the CPU oracle port of the reference algorithm
             (oracle/krylov_oracle.py, numpy/OpenBLAS on all host cores):
             configs 1-2 one full call per step; configs 3-5 a row sample of
             the configuration's own rows (host-rebuilt, see `sample`) run
             through the whole call, scaled to the full matrix.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = ("GK steps/s & time to top-k SVD; A·v+Aᵀu HBM GB/s vs roofline "
          "at 1/2/4/8 GPU")
UNIT = "GK steps/s"
FALLBACK_HBM_GBS = 6650.0
REF_SAMPLE_ROWS = 8192  # rows of the CPU sample for device-generated configs
DEFAULT_CONFIG = 4


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3,
                    help="end-to-end calls timed (each uploads the whole matrix)")
    ap.add_argument("--sample-rows", type=int, default=REF_SAMPLE_ROWS)
    return ap.parse_args(argv)


def workload(cfg_id):
    from paper_2104_10785_b200 import synth

    call = dict(synth.BASELINE_CALLS[cfg_id])
    if cfg_id == 1:
        W = dict(name="config1: fsvd k=30 r=10 eps=1e-10 of 2000x1000 f64 "
                 "(U diag(10^(-4(i-1)/999)) V^T, seed 0)", m=2000, n=1000, esize=8,
                 source="host")
    elif cfg_id == 2:
        W = dict(name="config2: estimate_rank eps=1e-6 relative of 20000x5000 f64 "
                 "(X Y^T + E, rank 137, seed 1)", m=20000, n=5000, esize=8, source="host")
    else:
        spec = synth.BASELINE_SPECS[cfg_id]
        what = "fsvd k=%d r=%d" % (call["k"], call["r"]) if call["kind"] == "fsvd" else \
            "estimate_rank eps=%g %s" % (call["eps"], call["mode"])
        W = dict(name=f"config{cfg_id}: {what} of {spec.m}x{spec.n} {spec.dtype} "
                 f"(P diag(s) Q^T + noise, rank {spec.rank}, {spec.spectrum} spectrum, "
                 f"seed {spec.seed}; generated in HBM)",
                 m=spec.m, n=spec.n, esize=4 if spec.dtype == "f32" else 8, source="device",
                 spec=spec)
    W.update(call)
    W["id"] = cfg_id
    return W


def config_dict(W):
    """The `config` object -- identical in both arms (same workload)."""
    a_bytes = W["m"] * W["n"] * W["esize"]
    return {"workload": W["name"], "m": W["m"], "n": W["n"],
            "A_storage": "f32" if W["esize"] == 4 else "f64",
            "l2": "A (%.0f MB) %s L2 (126 MB): no flush needed" % (
                a_bytes / 1e6, ">" if a_bytes > 126e6 else "<=")
            if a_bytes > 126e6 else "A (%.0f MB) <= L2 (126 MB): L2-resident" % (a_bytes / 1e6)}


def host_matrix(W, out=None):
    from paper_2104_10785_b200 import synth

    if W["id"] == 1:
        A = synth.config1_matrix(seed=0)
        if out is not None:
            out[...] = A
            return out
        return A
    return synth.config2_matrix(seed=W["seed"], out=out)


def call(K, W, A):
    """One bench step through the public API; returns (GK iterations, D2H bytes)."""
    if W["kind"] == "fsvd":
        psvd = K.fsvd(A, k=W["k"], r=W["r"],
                      cfg=K.BidiagConfig(k_max=W["k"], eps=W["eps"], seed=W["seed"]))
        fsvd_mod = sys.modules["paper_2104_10785_b200.fsvd"]

        # k' = the GK iterations the run performed (k unless it broke down)
        return fsvd_mod.last_k_prime, psvd.sigma.nbytes + psvd.U.nbytes + psvd.V.nbytes
    rep = K.estimate_rank(A, eps=W["eps"], mode=W["mode"], cfg=K.BidiagConfig(k_max=1, seed=W["seed"]))
    return rep.k_prime, 8 * (2 * rep.k_prime + 1)


def stage_breakdown(K, W, op, ctx):
    """One call of the entry point split into its stages, each timed on the
    host with a device sync after it (every rank runs it: the GK loop is
    collective); the same pieces fsvd / estimate_rank chain."""
    import ctypes as C

    from paper_2104_10785_b200 import _lib
    from paper_2104_10785_b200.bidiag import run_gk
    from paper_2104_10785_b200.fsvd import _gram, symtridiag_eig

    if W["kind"] == "fsvd":
        cfg = K.BidiagConfig(k_max=W["k"], eps=W["eps"], seed=W["seed"])
    else:
        cfg = K.BidiagConfig(k_max=min(W["m"], W["n"]), seed=W["seed"])
    ctx.sync()
    t0 = time.perf_counter()
    run = run_gk(op, cfg)
    ctx.sync()
    t1 = time.perf_counter()
    try:
        out = {"gk_loop": 1e3 * (t1 - t0), "gk_steps": run.k_prime}
        if W["kind"] != "fsvd":
            _lib.bidiag_sv2(run.alphas, run.betas)
            out["spectral"] = 1e3 * (time.perf_counter() - t1)
            return out
        theta, G = symtridiag_eig(_gram(run.alphas, run.betas))
        t2 = time.perf_counter()
        take = min(W["r"], run.k_prime)
        sig = np.ascontiguousarray(np.sqrt(np.maximum(theta[:take], 0.0)))
        Gt = np.ascontiguousarray(G[:, :take].T)
        Ub = np.empty((take, op.m_local))
        Vb = np.empty((take, W["n"]))
        good = C.c_int()
        _lib.check(_lib.load_library().ksvd_ritz(run.handle, _lib.dptr(Gt), _lib.dptr(sig),
                                                take, 1, _lib.dptr(Ub), _lib.dptr(Vb),
                                                C.byref(good)))
        ctx.sync()
        t3 = time.perf_counter()
        out.update({"spectral": 1e3 * (t2 - t1), "ritz_u_recovery_and_download": 1e3 * (t3 - t2)})
        return out
    finally:
        run.free()


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, device):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if mask & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=host_cores())
    except Exception:  # noqa: BLE001
        return host_cores()


# ----------------------------------------------------------------- CPU baseline
def _right_cgs_seconds(n, steps, reorth=2):
    """Seconds of the right-side CGS2 of `steps` GK steps (n-long vectors
    against the replicated right basis, bidiag.py:171-172): the part of a
    GK step that does NOT scale with the row count.  Same numpy operations
    on a C-order n x steps basis as the oracle."""
    rng = np.random.default_rng(0)
    right = np.linalg.qr(rng.standard_normal((n, steps)))[0].copy(order="C")
    z = rng.standard_normal(n)
    t0 = time.perf_counter()
    for i in range(1, steps):
        v = z
        for _ in range(reorth):
            v = v - right[:, :i] @ (right[:, :i].T @ v)
        float(np.linalg.norm(v))
    return time.perf_counter() - t0


class CpuSample:
    """The CPU reference (the oracle port) on a bounded sample of the
    workload.  Host configs: one full call on the config matrix.  Generated
    configs: S rows of the configuration's OWN rows (host rebuild of the
    generator: identical factor Gaussians and noise stream, numpy
    CholeskyQR2), through the whole reference call with the full call's
    iteration count; the m-proportional stages (products, left CGS2, U
    recovery and filter) are scaled by m / S, the n-sized ones (right CGS2,
    spectral stage, V = P G) are counted once."""

    def __init__(self, W, A_host=None, sample_rows=REF_SAMPLE_ROWS):
        self.W = W
        self.A = A_host
        if W["source"] == "device":
            from oracle.generated import host_generated_rows

            S = min(sample_rows, W["m"])
            r0 = (W["m"] - S) // 2
            t0 = time.perf_counter()
            rows = host_generated_rows(W["spec"], r0, S)
            self.A = rows(r0, r0 + S)
            self.rows_s = S
            self.build_s = time.perf_counter() - t0
            self.steps = W["k"] if W["kind"] == "fsvd" else W["expected_kprime"]
            self.right_s = None
        elif self.A is None:
            self.A = host_matrix(W)

    def run(self):
        """Returns (GK steps/s of the full call, description, seconds of CPU work)."""
        from oracle import krylov_oracle as O

        W = self.W
        if W["source"] == "host":
            t0 = time.perf_counter()
            if W["kind"] == "fsvd":
                O.fsvd_oracle(self.A, W["k"], W["r"], eps=W["eps"], seed=W["seed"])
                dt = time.perf_counter() - t0
                return W["k"] / dt, "one full oracle fsvd call on the config matrix", dt
            # the whole reference call (GK loop to breakdown + the Gram eigenvalues
            # + the count); a loop truncated early would omit the CGS2 cost that
            # grows with the step
            rep = O.rank_oracle(self.A, eps=W["eps"], mode=W["mode"], seed=W["seed"])
            dt = time.perf_counter() - t0
            return (rep.k_prime / dt, "one full oracle estimate_rank call on the config matrix "
                    f"(k' {rep.k_prime}, rank {rep.rank})", dt)
        m, n, S, k = W["m"], W["n"], self.rows_s, self.steps
        if self.right_s is None:
            self.right_s = _right_cgs_seconds(n, k)
        tm = {}
        t0 = time.perf_counter()
        if W["kind"] == "fsvd":
            O.fsvd_oracle(self.A, k, W["r"], eps=W["eps"], seed=W["seed"], timings=tm)
            scaled = tm["gk"] - self.right_s + tm["ritz_u"]
            once = self.right_s + tm["spectral"] + tm["ritz_v"]
        else:
            O.rank_oracle(self.A, eps=W["eps"], mode=W["mode"], seed=W["seed"], gk_eps=0.0,
                          k_max=k, timings=tm)
            scaled = tm["gk"] - self.right_s
            once = self.right_s + tm["spectral"]
        dt = time.perf_counter() - t0
        full = (m / S) * max(scaled, 0.0) + once
        desc = (f"oracle {W['kind']} call on rows [{(m - S) // 2}, {(m - S) // 2 + S}) of the "
                f"config's own matrix (host rebuild, f64), {k} GK steps (the full call's count), "
                f"{S}x{n}; m-proportional stages x {m / S:.1f} ({scaled:.2f} s), right CGS2 "
                f"+ spectral + V = P G once ({once:.2f} s) -> {full:.1f} s per full call")
        return k / full, desc, dt


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy)"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_from_profiles(cfg_id):
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()).get(f"config{cfg_id}")
    except Exception:  # noqa: BLE001
        return None


# --------------------------------------------------------------------------- arms
def run_reference(args, rank, world):
    """Reference arm: the oracle port of the reference on the host CPU (rank 0)."""
    if rank != 0:
        return
    W = workload(args.config)
    smp = CpuSample(W, sample_rows=args.sample_rows)
    vals, secs, desc = [], [], ""
    for i in range(args.warmup + args.steps):
        v, desc, dt = smp.run()
        if i >= args.warmup:
            vals.append(v)
            secs.append(dt)
    val = statistics.fmean(vals)
    cores = blas_threads()
    # one step = one (estimated, for the generated configs) full reference call
    ms_call = 1e3 * (statistics.fmean(secs) if W["source"] == "host" else smp.steps / val)
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_call,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference", "config": config_dict(W),
        "parallelism": "host cpu (%d BLAS threads)" % cores,
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": desc},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "effective_GBps": 2.0 * W["m"] * W["n"] * 8 * val / 1e9,
    }
    if W["source"] == "device":
        line["cpu_sample_build_s"] = smp.build_s
    emit(line)


def run_ours(args, rank, world, dist):
    import paper_2104_10785_b200 as K
    from paper_2104_10785_b200 import _lib, synth
    from paper_2104_10785_b200.dist import init_distributed

    ctx = init_distributed() if world > 1 else _lib.get_context()
    W = workload(args.config)
    m, n, es = W["m"], W["n"], W["esize"]

    def barrier():
        ctx.sync()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ingest = {}
    A_host = None
    barrier()
    t0 = time.perf_counter()
    if W["source"] == "host":
        A_host = host_matrix(W)
        t1 = time.perf_counter()
        op = K.DeviceMatrix.from_host(A_host)
        ctx.sync()
        ingest.update(host_build_s=t1 - t0, upload_s=time.perf_counter() - t1)
    else:
        op = synth.generate(W["spec"])
        ctx.sync()
        ingest["generate_s"] = max_over_ranks(time.perf_counter() - t0)
        ingest["generate_GBps"] = m * n * es / ingest["generate_s"] / 1e9
    m_local = op.m_local

    # ---- value: device-resident A ----
    for _ in range(args.warmup):
        call(K, W, op)
    barrier()
    ctx.reset_stats()
    kps = []
    with ClockSampler(ctx.device) as clk:
        ctx.mark(0)
        for _ in range(args.steps):
            kp, _ = call(K, W, op)
            kps.append(kp)
        ctx.mark(1)
        barrier()
    ms = max_over_ranks(ctx.elapsed_ms(0, 1))
    launches = ctx.launch_count()
    gk_steps = sum(kps)
    value = gk_steps / (ms / 1e3)
    eff_gbps = 2.0 * m * n * es * gk_steps / (ms / 1e3) / 1e9

    # ---- roofline: profiled repeat of the same calls ----
    barrier()
    ctx.reset_stats()
    ctx.set_profiling(True)
    for _ in range(max(1, min(args.steps, 2 if W["source"] == "device" else args.steps))):
        call(K, W, op)
    ctx.set_profiling(False)
    stats = {c: ctx.kernel_stats(c) for c in range(6)}
    barrier()
    bytes_launch = float(m_local) * n * es
    nn, msn = stats[0]
    nt, mst = stats[1]
    peak, peak_src = peak_hbm()
    per_kernel = {}
    for name, (cnt, kms) in (("gemv_n", stats[0]), ("gemv_t", stats[1])):
        if cnt:
            per_kernel[name] = {"launches": cnt, "avg_us": 1e3 * kms / cnt,
                                "GBps": bytes_launch / (kms / cnt / 1e3) / 1e9}
    achieved = (bytes_launch * (nn + nt)) / ((msn + mst) / 1e3) / 1e9 if nn + nt else 0.0
    kernel_desc = "gemv_n + gemv_t (A-streaming passes)"
    nr_, msr = stats[5]
    if nr_ and not nn + nt:
        # small matrix: the whole loop is one kernel with A in shared memory;
        # algorithmic bytes = 2 m n bytes per GK step over its duration
        steps_prof = kps[0] if kps else 0
        achieved = 2.0 * bytes_launch * steps_prof * nr_ / (msr / 1e3) / 1e9
        per_kernel["gk_resident"] = {"launches": nr_, "avg_us": 1e3 * msr / nr_,
                                     "GBps": achieved, "steps_per_launch": steps_prof}
        kernel_desc = ("k_gk_resident: whole GK loop, A resident in shared memory "
                       "(algorithmic 2*m*n*bytes per step / kernel time; latency-bound)")
    tot_prof = sum(v[1] for v in stats.values())
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": traffic_from_profiles(args.config),
        "kernel": kernel_desc, "peak_source": peak_src,
        "bytes_per_launch": bytes_launch, "per_kernel": per_kernel,
        "share_of_device_time": {k: v[1] / tot_prof for k, v in
                                 zip(["gemv_n", "gemv_t", "cgs", "other", "finalize",
                                      "gk_resident"], stats.values())} if tot_prof else None,
        "frac_of_nominal_8TBps": achieved / 8000.0,
        "frac_of_measured_read_7264GBps": achieved / 7263.6,
    }

    # ---- stages of one call (GK loop, spectral stage, Ritz/U
    # recovery reported separately): host wall time with a sync after each
    stages = stage_breakdown(K, W, op, ctx)
    barrier()

    # ---- config 1 as BASELINE words it: top-10 to convergence tol 1e-10 with
    # Krylov dimension 30 -- the restarted mode (the
    # reference has no restarts, so its call above stops unconverged)
    converged = None
    if args.config == 1 and world == 1:
        s_true = 10.0 ** (-4.0 * np.arange(W["n"]) / (W["n"] - 1))
        rcfg = K.BidiagConfig(k_max=30, seed=W["seed"])
        K.fsvd_restarted(op, 10, k=30, tol=1e-10, cfg=rcfg)
        ctx.sync()
        ctx.mark(4)
        reps = 10
        for _ in range(reps):
            ps, info = K.fsvd_restarted(op, 10, k=30, tol=1e-10, cfg=rcfg)
        ctx.mark(5)
        ctx.sync()
        converged = {
            "call": "fsvd_restarted(A, r=10, k=30, tol=1e-10) (thick Ritz restarts)",
            "ms": ctx.elapsed_ms(4, 5) / reps, "restarts": info.restarts,
            "gk_steps": info.gk_steps, "converged": info.converged,
            "max_sigma_relerr_vs_exact": float(np.max(np.abs(ps.sigma - s_true[:10])
                                                      / s_true[:10])),
            "max_residual_over_sigma1": float(np.max(info.residuals) / ps.sigma[0]),
        }

    # ---- e2e through the public API, from a plain host copy of this rank's rows ----
    e2e = None
    if not args.no_e2e:
        if A_host is None:
            t0 = time.perf_counter()
            A_local = op.to_dense()
            ingest["download_s"] = time.perf_counter() - t0
        else:
            A_local = np.ascontiguousarray(A_host[op.row0:op.row0 + m_local])
        row0 = op.row0
        op.free()
        del op
        ctx.release_pool()

        up_s = []

        def e2e_call():
            # DeviceMatrix.from_host + the entry point + the results on the host
            t0 = time.perf_counter()
            dm = K.DeviceMatrix.from_host(A_local, rows_are_local=True, m_global=m, row0=row0)
            up_s.append(time.perf_counter() - t0)  # from_host returns after the upload
            try:
                return call(K, W, dm)
            finally:
                dm.free()

        e2e_call()
        barrier()
        t_e2e, kps_e2e, d2h = [], [], 0
        for _ in range(max(1, args.e2e_steps)):
            ctx.mark(2)
            kp, nb = e2e_call()
            ctx.mark(3)
            ctx.sync()
            t_e2e.append(ctx.elapsed_ms(2, 3))
            kps_e2e.append(kp)
            d2h = nb
        barrier()
        e_ms = max_over_ranks(sum(t_e2e))
        h2d = int(A_local.nbytes + m_local * 8)
        e2e = {"value": sum(kps_e2e) / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms / len(t_e2e),
               "steps": len(t_e2e),
               "kind": "plain numpy A (pageable) uploaded every step through "
                       "DeviceMatrix.from_host (pinned staging inside libksvd), then the "
                       "entry point and the result read-back"}
        ingest["upload_s"] = statistics.median(up_s[1:])
        ingest["upload_GBps"] = A_local.nbytes / ingest["upload_s"] / 1e9
        del A_local

    # ---- CPU baseline (rank 0, N=1), after the GPU measurements: OpenBLAS's
    # spinning worker threads would otherwise steal the cores of the e2e upload ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        smp = CpuSample(W, A_host, sample_rows=args.sample_rows)
        v, desc, dt = smp.run()
        cpu = {"value": v, "unit": UNIT, "cores": blas_threads(), "kind": "port",
               "sample": desc, "seconds": dt}
        del smp
        if converged is not None:
            from oracle.restarted import restarted_oracle

            t0 = time.perf_counter()
            restarted_oracle(A_host, 10, 30, tol=1e-10, seed=W["seed"])
            converged["cpu_port_ms"] = 1e3 * (time.perf_counter() - t0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if es == 8 else "f64 (f32 storage of A)", "data": "synthetic",
            "config": config_dict(W),
            "parallelism": f"row-shard x{world} (NCCL)" if world > 1 else "single GPU",
            "time_to_result_s": ms / args.steps / 1e3,
            "gk_steps_per_call": kps[0] if kps else None,
            "effective_GBps": eff_gbps,
            # 2 m n bytes per GK step over the whole call vs the aggregate HBM peak
            "effective_frac_of_hbm_peak": eff_gbps / (peak * world),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "ingest": ingest,
            "gpu_launches": launches,
            "converged_top_k": converged,
            "stages_ms": stages,
            "clocks": clk.summary(),
        }
        emit(line)


_JSON_OUT = None


def emit(line):
    """The one JSON line on the process's real stdout (see main)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


# ------------------------------------------------------------------- launcher
def visible_gpus() -> int:
    from paper_2104_10785_b200 import _lib

    return _lib.device_count()


def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def rank_envs(n: int, port: int, base: dict | None = None) -> list[dict]:
    """The environment of each of the N ranks bench.py starts itself (the
    variables torchrun would set), NCCL's INFO log on stderr for N > 1."""
    base = dict(os.environ if base is None else base)
    out = []
    for r in range(n):
        env = dict(base)
        env.update(RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   GROUP_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        if n > 1:
            env.setdefault("NCCL_DEBUG", "INFO")
        out.append(env)
    return out


def launch(n: int, argv, script: str | None = None, check_gpus: bool = True) -> int:
    """Start n ranks of `script` (default: this file; one process per GPU)
    with the torchrun environment, rank 0 writing to the real stdout; wait
    for all of them.  Returns the first non-zero exit code (the other ranks
    are then terminated, they would wait on the failed one forever)."""
    if n < 1:
        print(f"bench.py: --gpus must be >= 1, got {n}", file=sys.stderr)
        return 2
    if check_gpus:
        have = visible_gpus()
        if have < n:
            print(f"bench.py: --gpus {n} but only {have} GPU(s) visible", file=sys.stderr)
            return 3
    script = str(Path(script or __file__).resolve())
    out0 = _JSON_OUT or sys.stdout
    procs = [subprocess.Popen([sys.executable, script, *argv], env=env,
                              stdout=out0 if r == 0 else sys.stderr, stderr=sys.stderr)
             for r, env in enumerate(rank_envs(n, free_port()))]
    rc = 0
    alive = set(range(n))
    while alive:
        for r in sorted(alive):
            code = procs[r].poll()
            if code is None:
                continue
            alive.discard(r)
            if code != 0 and rc == 0:
                rc = code
                for o in alive:
                    procs[o].terminate()
        time.sleep(0.1)
    return rc


def main():
    global _JSON_OUT
    # Library chatter (NCCL prints its version banner and INFO lines to fd 1
    # when its debug level asks for it) must not precede the JSON line the
    # driver parses: fd 1 is pointed at stderr for the whole run and the
    # line goes to a duplicate of the original stdout.
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    argv = sys.argv[1:]
    args = parse(argv)
    if "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":  # host CPU only: rank 0 of a notional N-rank job
            run_reference(args, 0, args.gpus)
            return 0
        return launch(args.gpus, argv)
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE {world} != --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        run_reference(args, rank, world)
        return 0
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
    run_ours(args, rank, world, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
