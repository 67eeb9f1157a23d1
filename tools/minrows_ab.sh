#!/bin/bash
# config-2 bench under CGS tile-geometry / reduction-mode settings
for e in KSVD_NONE=1 KSVD_CGS_MINROWS=64 KSVD_CGS_MINROWS=128 KSVD_CGS_MINROWS=96 "KSVD_CGS_MINROWS=128 KSVD_RED_MAX=6000" KSVD_NONE=1; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mr.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/mr.json'));print('$e', round(d['value'],1), round(d['ms_per_step'],3))"
done
