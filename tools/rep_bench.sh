#!/bin/bash
# default config-2 bench, repeated (run-to-run spread)
for r in 1 2 3; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rb.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/rb.json'));print('run $r', round(d['value'],1), round(d['ms_per_step'],3), d['clocks'])"
done
