#!/bin/bash
# k_gemv_n (CTA-reduced) in the library: GPU suite, then config 2 and 4 benches vs the pre-change build
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02e; mkdir -p $O
timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
for i in 1 2; do
  KSVD_LIB_PATH=tools/ab/libksvd_gemvn2.so timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/c2_old_$i.json 2>> $O/ab.err
  timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/c2_new_$i.json 2>> $O/ab.err
done
KSVD_LIB_PATH=tools/ab/libksvd_gemvn2.so timeout 900 python bench.py --config 4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $O/c4_old.json 2>> $O/ab.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $O/c4_new.json 2>> $O/ab.err
for f in $O/c*.json; do echo "$f $(python -c "
import json; d=json.loads(open('$f').read()); r=d['roofline']
print(round(d['value'],2), {k: round(v['GBps']) for k, v in r['per_kernel'].items()}, round(r['share_of_device_time']['cgs'],4), d['clocks']['sm_mhz'])")"; done
