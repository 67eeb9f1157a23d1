#!/bin/bash
# paired step: redundant vs distributed reductions (KSVD_RED_MAX) on config 2
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/redmax; mkdir -p $O
for i in 1 2; do
for rm in 0 2368 8000 100000000; do
  KSVD_RED_MAX=$rm timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/rm${rm}_$i.json 2>> $O/err.txt
  python -c "
import json; d=json.load(open('$O/rm${rm}_$i.json')); print('red_max $rm', round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['share_of_device_time']['cgs'],4), d['clocks']['sm_mhz'])"
done
done
