#!/bin/bash
# config-2 bench: PDL trigger placement (bit 0 gemv early, bit 1 CGS early)
for e in KSVD_PDL_TRIG=1 KSVD_PDL_TRIG=3 KSVD_PDL_TRIG=0 KSVD_PDL_TRIG=1 KSVD_PDL_TRIG=3; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tr.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/tr.json'));print('$e', round(d['value'],1), round(d['ms_per_step'],3))"
done
