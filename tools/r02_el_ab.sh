#!/bin/bash
# paired step: bases loaded / written L2::evict_last (default) vs default priority
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/el; mkdir -p $O
for i in 1 2 3; do
for v in 0 1; do
  KSVD_PAIR_EVICT_LAST=$v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_el${v}_$i.json 2>> $O/err.txt
  python -c "
import json; d=json.load(open('$O/c2_el${v}_$i.json')); pk=d['roofline']['per_kernel']; sh=d['roofline']['share_of_device_time']
print('config 2 evict_last $v', round(d['value'],1), round(d['ms_per_step'],3), {k: round(v['GBps']) for k,v in pk.items()}, 'cgs', round(sh['cgs'],4), d['clocks']['sm_mhz'])"
done
done
