"""Host wall-time breakdown of one fsvd call on a BASELINE config (3 or 4):
GK loop, host eigensolver, ksvd_ritz (V = P G, U = A V / sigma, U filter,
sign fix, download of U and V)."""
import argparse
import ctypes as C
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import _lib, synth
from paper_2104_10785_b200.bidiag import run_gk
from paper_2104_10785_b200.fsvd import _gram, symtridiag_eig

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
a = ap.parse_args()
call = synth.BASELINE_CALLS[a.config]
op = synth.generate(synth.BASELINE_SPECS[a.config])
ctx = _lib.get_context()
cfg = K.BidiagConfig(k_max=call["k"], eps=call["eps"], seed=call["seed"])
for it in range(3):
    ctx.sync()
    t0 = time.perf_counter()
    run = run_gk(op, cfg)
    ctx.sync()
    t1 = time.perf_counter()
    theta, G = symtridiag_eig(_gram(run.alphas, run.betas))
    t2 = time.perf_counter()
    take = call["r"]
    sig = np.sqrt(theta[:take])
    Gt = np.ascontiguousarray(G[:, :take].T)
    Ub = np.empty((take, op.m_local))
    Vb = np.empty((take, op.shape[1]))
    good = C.c_int()
    _lib.check(_lib.load_library().ksvd_ritz(run.handle, _lib.dptr(Gt), _lib.dptr(sig), take, 1,
                                            _lib.dptr(Ub), _lib.dptr(Vb), C.byref(good)))
    ctx.sync()
    t3 = time.perf_counter()
    run.free()
    t4 = time.perf_counter()
    K.fsvd(op, k=call["k"], r=call["r"], cfg=cfg)
    ctx.sync()
    t5 = time.perf_counter()
    print(f"config {a.config} call {it}: run_gk {1e3*(t1-t0):.1f} ms, eig {1e3*(t2-t1):.2f} ms, "
          f"ritz+download {1e3*(t3-t2):.1f} ms (U {Ub.nbytes/1e6:.0f} MB), free {1e3*(t4-t3):.2f} ms"
          f" | fsvd {1e3*(t5-t4):.1f} ms", flush=True)
