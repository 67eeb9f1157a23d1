"""Config-1 call breakdown: GK (resident kernel) vs the rest of fsvd."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import _lib, synth
from paper_2104_10785_b200.bidiag import run_gk

op = K.DeviceMatrix.from_host(synth.config1_matrix(seed=0))
ctx = _lib.get_context()
cfg = K.BidiagConfig(k_max=30, eps=1e-10, seed=0)
for _ in range(5):
    K.fsvd(op, k=30, r=10, cfg=cfg)
ctx.sync()
N = 50
t = time.perf_counter()
for _ in range(N):
    K.fsvd(op, k=30, r=10, cfg=cfg)
ctx.sync()
t_call = (time.perf_counter() - t) / N
t = time.perf_counter()
for _ in range(N):
    run = run_gk(op, cfg)
    run.free()
ctx.sync()
t_gk = (time.perf_counter() - t) / N
ctx.set_profiling(True)
ctx.reset_stats()
for _ in range(N):
    K.fsvd(op, k=30, r=10, cfg=cfg)
ctx.set_profiling(False)
names = ["gemv_n", "gemv_t", "cgs/resident", "other", "finalize"]
stats = {names[c]: ctx.kernel_stats(c) for c in range(5)}
print(f"fsvd call {1e3 * t_call:.3f} ms, run_gk alone {1e3 * t_gk:.3f} ms")
for k, (cnt, ms) in stats.items():
    if cnt:
        print(f"  {k:14s} {cnt / N:6.1f} launches/call {1e3 * ms / N:8.1f} us/call")
from paper_2104_10785_b200.bidiag import _start_vector
t = time.perf_counter()
for _ in range(N):
    _start_vector(cfg, 2000)
print(f"  start vector (host numpy) {1e6 * (time.perf_counter() - t) / N:.1f} us")
