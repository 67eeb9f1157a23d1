#!/bin/bash
# config-2 bench: event pacing (default) vs progress-word pacing
for e in KSVD_NONE=1 KSVD_PACE=spin KSVD_NONE=1 KSVD_PACE=spin; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pc.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/pc.json'));print('$e', round(d['value'],1), round(d['ms_per_step'],3))"
done
