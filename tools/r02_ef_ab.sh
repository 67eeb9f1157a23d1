#!/bin/bash
# A-streaming loads with an L2 evict_first policy (KSVD_A_EVICT_FIRST=1) vs evict_normal, same box
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ef; mkdir -p $O
for c in 2 3 4; do
for i in 1 2; do
for ef in 0 1; do
  KSVD_A_EVICT_FIRST=$ef timeout 900 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > $O/c${c}_ef${ef}_$i.json 2>> $O/err.txt
  python -c "
import json; d=json.load(open('$O/c${c}_ef${ef}_$i.json')); pk=d['roofline']['per_kernel']; sh=d['roofline']['share_of_device_time']
print('config $c ef $ef', round(d['value'],2), round(d['ms_per_step'],3), {k: round(v['GBps']) for k,v in pk.items()}, 'cgs', round(sh['cgs'],4), d['clocks']['sm_mhz'])"
done
done
done
