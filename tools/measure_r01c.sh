#!/bin/bash
# Late round-1 refresh: bench lines for configs 1-5, the config-2 launch list
# of the bench command, ncu --set full of the step kernels at config 2.
mkdir -p gpurun_out
bash tools/bench_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 2 --warmup 1 \
  --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench_c2.log 2>&1
python tools/launch_summary.py gpurun_out/launches_bench_c2.csv > gpurun_out/launches_config2.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gemv_n2|k_gemv_t2|k_cgs2_tile2" -s 200 -c 4 -o gpurun_out/prof_c2_r01c -f \
  python tools/one_call.py --config 2 --calls 1 > gpurun_out/ncu_full_c2.log 2>&1
echo done
