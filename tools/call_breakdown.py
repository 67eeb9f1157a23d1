"""Host-side time breakdown of one estimate_rank call (config 2)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import _lib, synth
from paper_2104_10785_b200.bidiag import run_gk
from paper_2104_10785_b200.fsvd import _gram

A = synth.config2_matrix(seed=1)
op = K.DeviceMatrix.from_host(A)
cfg = K.BidiagConfig(k_max=5000, seed=1)
ctx = _lib.get_context()
for it in range(4):
    ctx.sync()
    t0 = time.perf_counter()
    run = run_gk(op, cfg)
    t1 = time.perf_counter()
    theta, _ = K.symtridiag_eig(_gram(run.alphas, run.betas), vectors=False)
    t2 = time.perf_counter()
    run.free()
    t3 = time.perf_counter()
    print(f"call {it}: run_gk {1e3*(t1-t0):.2f} ms, eig {1e3*(t2-t1):.2f} ms, free {1e3*(t3-t2):.2f} ms, k' {run.k_prime}")
