#!/bin/bash
# same-box A/B on config 2: pre-prune library vs cluster sizes / min rows per CTA
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02d; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/$name.json 2>> $O/ab.err; }
for i in 1 2; do
  run old_$i KSVD_LIB_PATH=tools/ab/libksvd_pre_prune.so
  run cs1_$i KSVD_CGS_CLUSTER=1
  run cs8_$i KSVD_CGS_CLUSTER=8
  run cs8_mr64_$i KSVD_CGS_CLUSTER=8 KSVD_CGS_MINROWS=64
  run cs1_mr64_$i KSVD_CGS_CLUSTER=1 KSVD_CGS_MINROWS=64
  run cs1_mr128_$i KSVD_CGS_CLUSTER=1 KSVD_CGS_MINROWS=128
  run old_mr64_$i KSVD_LIB_PATH=tools/ab/libksvd_pre_prune.so KSVD_CGS_MINROWS=64
done
for f in $O/*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read()); print(round(d['value'],1), round(d['roofline']['share_of_device_time']['cgs'],4), d['clocks']['sm_mhz'])")"; done
