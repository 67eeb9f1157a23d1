KSVD_DEBUG_HOST=1 KSVD_PHASE_TIMES=1 timeout 600 python -c "
import sys, time; sys.path.insert(0,'.')
import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth, _lib
from paper_2104_10785_b200.bidiag import run_gk
op = synth.generate(synth.BASELINE_SPECS[5])
ctx = _lib.get_context()
for it in range(2):
    ctx.sync(); t0=time.perf_counter()
    run = run_gk(op, K.BidiagConfig(k_max=20000, eps=1e-8, seed=4))
    t1=time.perf_counter()
    th = _lib.bidiag_sv2(run.alphas, run.betas); t2=time.perf_counter()
    run.free(); ctx.sync(); t3=time.perf_counter()
    print('run_gk %.3f s  sv2 %.4f s  free %.4f s  kp %d' % (t1-t0, t2-t1, t3-t2, run.k_prime), flush=True)
" > gpurun_out/dbg_c5.log 2>&1
