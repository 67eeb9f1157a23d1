#!/bin/bash
# A/B of the row-streamed persistent kernel (KSVD_ROWS) on config 2 + phases
KSVD_ROWS=1 KSVD_PHASE_TIMES=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth
from paper_2104_10785_b200.bidiag import run_gk
op = K.DeviceMatrix.from_host(synth.config2_matrix(seed=1))
for it in range(2):
    run = run_gk(op, K.BidiagConfig(k_max=5000, seed=1)); print('kp', run.k_prime); run.free()
" 2>&1 | grep -E "phases|kp|Error|error" | tail -4
for r in 1 2; do
  for st in 0 1; do
    KSVD_ROWS=$st timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rab.out 2>gpurun_out/rab.err
    python -c "import json; d=json.load(open('gpurun_out/rab.out')); print('rows $st', round(d['value'],1), round(d['ms_per_step'],3), d['gk_steps_per_call'], d['gpu_launches'])" || tail -3 gpurun_out/rab.err
  done
done
