#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02f; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_restart.py -x -q > $O/restart.log 2>&1; tail -2 $O/restart.log
for i in 1 2; do
  KSVD_LIB_PATH=tools/ab/libksvd_gemvn2.so timeout 900 python bench.py --config 4 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $O/c4_old_$i.json 2>> $O/ab.err
  timeout 900 python bench.py --config 4 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $O/c4_new_$i.json 2>> $O/ab.err
done
for f in $O/c*.json; do echo "$f $(python -c "
import json; d=json.loads(open('$f').read()); r=d['roofline']
print(round(d['value'],2), round(d['ms_per_step']), {k: round(v['GBps']) for k, v in r['per_kernel'].items()}, round(d['stages_ms']['gk_loop']), d['clocks']['sm_mhz'])")"; done
