#!/bin/bash
# A/B two builds of libksvd on the same box: ./tools/ab.sh <libA> <libB> [config] [reps]
A=$1; B=$2; CFG=${3:-2}; REPS=${4:-3}
for r in $(seq $REPS); do
  for L in $A $B; do
    KSVD_LIB_PATH=$L python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.out 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.out')); print('$L'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],3), {k:round(v['GBps']) for k,v in d['roofline']['per_kernel'].items()})"
  done
done
