#!/bin/bash
# k_gemv_n: named-barrier CTA row sums (KSVD_GEMVN_NB=1) vs __syncthreads, same box
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/nb; mkdir -p $O
KSVD_GEMVN_NB=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log; tail -2 $O/tests.log
for c in 2 4; do
for i in 1 2; do
for nb in 0 1; do
  KSVD_GEMVN_NB=$nb timeout 900 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > $O/c${c}_nb${nb}_$i.json 2>> $O/err.txt
  python -c "
import json; d=json.load(open('$O/c${c}_nb${nb}_$i.json')); pk=d['roofline']['per_kernel']
print('config $c nb $nb', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['GBps']) for k,v in pk.items()}, d['clocks']['sm_mhz'])"
done
done
done
