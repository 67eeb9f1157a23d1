#!/bin/bash
# k_cgs2_pair triggering the next product after its last grid round (KSVD_PAIR_TRIG=1) vs at exit
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/trig; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "paired or golden" 2>&1 | tail -1
KSVD_PAIR_TRIG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "paired or golden" 2>&1 | tail -1
for i in 1 2 3; do
for v in 0 1; do
  KSVD_PAIR_TRIG=$v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_t${v}_$i.json 2>> $O/err.txt
  python -c "
import json; d=json.load(open('$O/c2_t${v}_$i.json')); pk=d['roofline']['per_kernel']; sh=d['roofline']['share_of_device_time']
print('config 2 trig $v', round(d['value'],1), round(d['ms_per_step'],3), {k: round(v['GBps']) for k,v in pk.items()}, 'cgs', round(sh['cgs'],4), d['clocks']['sm_mhz'])"
done
done
