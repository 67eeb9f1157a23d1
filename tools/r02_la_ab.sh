#!/bin/bash
# lookahead GK step: parity suites first (bounded), then a same-box A/B
# against the serialised step (KSVD_LOOKAHEAD=0) on configs 2 and 3
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/la; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -5 $O/tests.log
for c in 2 3; do
  for i in 1 2; do
    KSVD_LOOKAHEAD=0 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/off_c${c}_$i.json 2>> $O/ab.err
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/on_c${c}_$i.json 2>> $O/ab.err
  done
done
for f in $O/off_c*.json $O/on_c*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],2), d['roofline']['share_of_device_time'].get('cgs'), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
