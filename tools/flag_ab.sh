#!/bin/bash
# config-2 bench: flag barrier (default) vs the flip barrier
for e in KSVD_NONE=1 KSVD_FLAG_BARRIER=0 KSVD_NONE=1 KSVD_FLAG_BARRIER=0; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fb.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/fb.json'));print('$e', round(d['value'],1), round(d['ms_per_step'],3))"
done
