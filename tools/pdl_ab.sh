#!/bin/bash
# A/B of programmatic dependent launch / trigger placement (1 GPU)
mkdir -p gpurun_out
run() {  # cfg pdl trig
  KSVD_PDL=$2 KSVD_PDL_TRIG=$3 timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $1 pdl $2 trig $3', round(d['value'],1), round(d['ms_per_step'],3))"
}
for cfg in ${CFGS:-2 1}; do
  for rep in 1 2; do
    run $cfg 0 3
    for trig in 0 1 2 3; do run $cfg 1 $trig; done
  done
done
