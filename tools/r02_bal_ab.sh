#!/bin/bash
# k_gemv_n balanced grid (last narrow chunk group with fewer, longer segments) vs uniform, same box
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/bal; mkdir -p $O
KSVD_RESIDENT=0 timeout 900 python -m pytest tests/test_gpu_fuzz.py::test_fuzz_vs_oracle tests/test_gpu_parity.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log; tail -2 $O/tests.log
for c in 4 3; do
for i in 1 2; do
for b in 0 1; do
  KSVD_GEMVN_BAL=$b timeout 900 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > $O/c${c}_b${b}_$i.json 2>> $O/err.txt
  python -c "
import json; d=json.load(open('$O/c${c}_b${b}_$i.json')); pk=d['roofline']['per_kernel']
print('config $c bal $b', round(d['value'],2), round(d['ms_per_step'],2), {k: (round(v['GBps']), round(v['avg_us'],1)) for k,v in pk.items()}, d['clocks']['sm_mhz'])"
done
done
done
