#!/bin/bash
# pacing events every 1 / 2 / 4 steps on config 2 (same box)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/pace; mkdir -p $O
for i in 1 2; do
for e in 1 2 4; do
  KSVD_PACE_EVERY=$e timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/e${e}_$i.json 2>> $O/err.txt
  python -c "
import json; d=json.load(open('$O/e${e}_$i.json')); print('every $e', round(d['value'],1), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done
done
