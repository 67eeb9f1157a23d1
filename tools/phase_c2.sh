#!/bin/bash
# CGS tile-kernel phase timing (CTA 0, globaltimer) on config 2; extra env
# settings to compare are passed as arguments (default: the library defaults)
for envs in "${@:-KSVD_NONE=1}"; do
env $envs KSVD_DEBUG_HOST=1 KSVD_PHASE_TIMES=1 timeout 600 python -c "
import sys, time; sys.path.insert(0,'.')
import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth, _lib
from paper_2104_10785_b200.bidiag import run_gk
op = K.DeviceMatrix.from_host(synth.config2_matrix(seed=1))
ctx = _lib.get_context()
for it in range(3):
    ctx.sync(); t0=time.perf_counter()
    run = run_gk(op, K.BidiagConfig(k_max=5000, seed=1))
    ctx.sync(); t1=time.perf_counter()
    print('[$envs] run_gk %.3f ms kp %d' % (1e3*(t1-t0), run.k_prime), flush=True)
    run.free()
" 2>&1 | grep -v "^\[ksvd\] gk host"
done
