#!/bin/bash
# round-2 validation pass: GPU tests, full-size parity, pre/post-prune A/B on
# config 2, the config-4 bench (both arms)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi0.csv
timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 1200 python -m pytest tests/test_gpu_fullsize_parity.py -x -q -rs > $O/fullsize_parity.log 2>&1; echo "rc=$?" >> $O/fullsize_parity.log
for i in 1 2; do
  KSVD_LIB_PATH=tools/ab/libksvd_pre_prune.so timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/ab_old_$i.json 2>> $O/ab.err
  timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/ab_new_$i.json 2>> $O/ab.err
done
timeout 1500 python bench.py --steps 3 --warmup 1 > $O/bench_c4.json 2> $O/bench_c4.err; echo "rc=$?" >> $O/bench_c4.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/ref_c4.json 2> $O/ref_c4.err; echo "rc=$?" >> $O/ref_c4.err
tail -3 $O/gpu_tests.log $O/fullsize_parity.log
