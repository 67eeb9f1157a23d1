#!/bin/bash
# A/B: 5-round k_cgs2_tile vs k_cgs2_tile2 at several redundant-reduce caps
run() {  # cfg sync redmax
  KSVD_CGS_SYNC=$2 KSVD_RED_MAX=$3 timeout 600 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $1 sync $2 redmax $3', round(d['value'],1), round(d['ms_per_step'],3), d['gk_steps_per_call'])"
}
for cfg in ${CFGS:-2 1}; do
  for rep in 1 2; do run $cfg 5 0; for rm in 0 2368 7104 14208 100000; do run $cfg 2 $rm; done; done
done
