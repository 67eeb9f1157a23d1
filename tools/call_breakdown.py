"""Host-side time breakdown of one estimate_rank call (config 2): the GK
loop (start vector, device loop, alpha/beta download), the rank path's
bidiagonal SVD, the run release."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import _lib, synth
from paper_2104_10785_b200.bidiag import _start_vector, run_gk

A = synth.config2_matrix(seed=1)
op = K.DeviceMatrix.from_host(A)
cfg = K.BidiagConfig(k_max=5000, seed=1)
ctx = _lib.get_context()
for it in range(4):
    ctx.sync()
    t0 = time.perf_counter()
    _start_vector(cfg, op.shape[0])
    ts = time.perf_counter()
    run = run_gk(op, cfg)
    t1 = time.perf_counter()
    theta = _lib.bidiag_sv2(run.alphas, run.betas)
    t2 = time.perf_counter()
    run.free()
    t3 = time.perf_counter()
    print(f"call {it}: start vector {1e3*(ts-t0):.2f} ms, run_gk {1e3*(t1-ts):.2f} ms, "
          f"bidiag_sv2 {1e3*(t2-t1):.2f} ms, free {1e3*(t3-t2):.2f} ms, k' {run.k_prime}")
    ctx.sync()
    t4 = time.perf_counter()
    rep = K.estimate_rank(op, eps=1e-6, mode="relative", cfg=cfg)
    ctx.sync()
    print(f"        estimate_rank {1e3*(time.perf_counter()-t4):.2f} ms, rank {rep.rank}")
