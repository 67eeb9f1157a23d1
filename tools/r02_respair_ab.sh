#!/bin/bash
# resident kernel: paired step (4 grid rounds) vs serialised (6); parity
# suites first, then config 1 bench lines both ways, one box
cd "${GRAFT_REPO_ROOT:-.}"
O=${OUT:-gpurun_out/respair}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py tests/test_gpu_restart.py tests/test_gpu_acceptance.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -4 $O/tests.log
for i in 1 2 3; do
  for v in "KSVD_RES_PAIR=0" "X=1"; do
    env $v timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/c1_${v%%=*}_$i.json 2>> $O/ab.err
  done
done
for f in $O/c1_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],4), d.get('converged_top_k'), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
KSVD_PHASE_TIMES=1 python tools/one_call.py --config 1 --calls 3 2>&1 | tail -4
KSVD_RES_PAIR=0 KSVD_PHASE_TIMES=1 python tools/one_call.py --config 1 --calls 3 2>&1 | tail -4
