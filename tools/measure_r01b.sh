#!/bin/bash
# Round-1 late measurement: bench lines for configs 1-5, config-2 launch
# list (the bench command itself), ncu --set full of the step kernels.
mkdir -p gpurun_out
bash tools/bench_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 2 --warmup 1 \
  --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench_c2.log 2>&1
python tools/one_call.py --config 2 --calls 1 > gpurun_out/plain_c2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gemv_n2|k_gemv_t2|k_cgs2_tile2" -s 40 -c 3 -o gpurun_out/prof_c2_r01b \
  python tools/one_call.py --config 2 --calls 1 > gpurun_out/ncu_full_c2.log 2>&1
echo done
