#!/bin/bash
# config-2 bench: redundant-reduction threshold of k_cgs2_tile2 (doubles per CTA)
for e in KSVD_RED_MAX=2368 KSVD_RED_MAX=1184 KSVD_RED_MAX=3552 KSVD_RED_MAX=4736 KSVD_RED_MAX=2368 KSVD_RED_MAX=0; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rm.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/rm.json'));print('$e', round(d['value'],1), round(d['ms_per_step'],3))"
done
