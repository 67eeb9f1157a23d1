#!/bin/bash
# A/B: multi-kernel vs global-load cooperative CGS2 for bases too large for tiles
for cfg in ${CFGS:-3}; do
  for g in 0 1 0 1; do
    KSVD_COOP_GLOBAL=$g timeout 900 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/cg.out 2>gpurun_out/cg.err
    python -c "import json; d=json.load(open('gpurun_out/cg.out')); print('cfg $cfg global $g', round(d['value'],2), round(d['ms_per_step'],1), {k: round(v,4) for k,v in d['roofline']['share_of_device_time'].items()})" || tail -3 gpurun_out/cg.err
  done
done
