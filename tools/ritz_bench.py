"""Ritz / restart contraction timing (k_basis_combine_dmma) on a config-3
sized basis: fsvd_restarted on the device-generated config-3 matrix with a
small basis, plus the ncu target for the tensor-pipe counters."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import _lib, synth

spec = synth.BASELINE_SPECS[3]
op = synth.generate(spec)
ctx = _lib.get_context()
for it in range(2):
    ctx.set_profiling(True)
    ctx.reset_stats()
    t = time.perf_counter()
    ps, info = K.fsvd_restarted(op, 20, k=60, tol=1e-10, cfg=K.BidiagConfig(k_max=60, seed=2))
    dt = time.perf_counter() - t
    ctx.set_profiling(False)
    n_o, ms_o = ctx.kernel_stats(3)
    print(f"restarted fsvd config 3: {dt:.3f} s, restarts {info.restarts}, steps {info.gk_steps}, "
          f"converged {info.converged}, sigma[:3] {ps.sigma[:3]}, other-kernels {n_o} launches "
          f"{ms_o:.2f} ms", flush=True)
