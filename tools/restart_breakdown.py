"""Host wall-time breakdown of fsvd_restarted on config 1 (r=10, k=30,
tol 1e-10): GK run, per-cycle info download, host dense SVD, device restart
(basis contraction + resumed loop), final Ritz bases."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import _lib, restart, synth

op = K.DeviceMatrix.from_host(synth.config1_matrix(seed=0))
ctx = _lib.get_context()
cfg = K.BidiagConfig(k_max=30, seed=0)
acc = {}
orig = {n: getattr(restart, n) for n in ("run_gk", "_info", "dense_svd")}
lib = _lib.load_library()
orig_restart = lib.ksvd_run_restart
orig_ritz = lib.ksvd_run_ritz_bases


def timed(name, f):
    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        ctx.sync()
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        return r
    return g


for n, f in orig.items():
    setattr(restart, n, timed(n, f))
for _ in range(3):
    K.fsvd_restarted(op, 10, k=30, tol=1e-10, cfg=cfg)
acc.clear()
N = 20
ctx.sync()
t0 = time.perf_counter()
for _ in range(N):
    ps, info = K.fsvd_restarted(op, 10, k=30, tol=1e-10, cfg=cfg)
ctx.sync()
tot = (time.perf_counter() - t0) / N
print(f"fsvd_restarted {1e3 * tot:.3f} ms/call, restarts {info.restarts}, steps {info.gk_steps}")
for k, v in acc.items():
    print(f"  {k:10s} {1e3 * v / N:.3f} ms/call")
