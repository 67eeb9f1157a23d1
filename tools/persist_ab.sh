#!/bin/bash
# config-2 bench: the 4-launch loop (default) vs the persistent step kernels
for e in KSVD_NONE=1 KSVD_ROWS=1 KSVD_STREAM=1 KSVD_NONE=1; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pa.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/pa.json'));print('$e', round(d['value'],1), round(d['ms_per_step'],3))"
done
