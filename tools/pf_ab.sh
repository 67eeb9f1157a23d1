#!/bin/bash
# A/B of the k_gemv_n2 prefetch plan on configs 3 and 4 (same box)
for cfg in ${CFGS:-4 3}; do
  for pf in 0 1; do
    KSVD_GEMVN_PF=$pf timeout 900 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/pf.out 2>gpurun_out/pf.err
    python -c "import json; d=json.load(open('gpurun_out/pf.out')); print('cfg $cfg pf $pf', round(d['value'],2), round(d['ms_per_step'],1), {k:round(v['GBps']) for k,v in d['roofline']['per_kernel'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pf.err
  done
done
