#!/bin/bash
# A/B: cooperative vs regular (custom barrier, PDL-overlappable) CGS launches
for r in 1 2 3; do
  for cl in 1 0; do
    KSVD_COOP_LAUNCH=$cl timeout 300 python bench.py --config ${CFG:-2} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cab.out 2>gpurun_out/cab.err
    python -c "import json; d=json.load(open('gpurun_out/cab.out')); print('coop_launch $cl', round(d['value'],1), round(d['ms_per_step'],3), d['gk_steps_per_call'])" || tail -3 gpurun_out/cab.err
  done
done
