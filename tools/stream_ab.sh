#!/bin/bash
# A/B of the persistent streaming kernel (KSVD_STREAM) on config 2
for r in 1 2; do
  for st in 0 1; do
    KSVD_STREAM=$st python bench.py --config ${CFG:-2} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sab.out 2>gpurun_out/sab.err
    python -c "import json; d=json.load(open('gpurun_out/sab.out')); print('stream $st', round(d['value'],1), round(d['ms_per_step'],3), d['gk_steps_per_call'], d['gpu_launches'])" || tail -3 gpurun_out/sab.err
  done
done
