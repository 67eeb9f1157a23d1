#!/bin/bash
# same-box A/B: working tree library vs tools/ab/libksvd_head.so (last commit) on config 2 (+ parity)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ab_head; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -x -q > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log; tail -2 $O/parity.log
for i in 1 2 3; do
  KSVD_LIB_PATH=tools/ab/libksvd_head.so timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/c2_head_$i.json 2>> $O/ab.err
  timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/c2_new_$i.json 2>> $O/ab.err
done
for f in $O/c2_*.json; do echo "$f $(python -c "
import json; d=json.loads(open('$f').read()); r=d['roofline']
print(round(d['value'],1), round(d['ms_per_step'],2), round(r['share_of_device_time']['cgs'],4), {k: round(v['GBps']) for k, v in r['per_kernel'].items()}, d['clocks']['sm_mhz'])")"; done
