#!/bin/bash
python tools/ritz_bench.py > gpurun_out/ritz_bench.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:"k_basis_combine_dmma|k_multi_rhs" -c 4 \
  -o gpurun_out/prof_ritz python tools/one_call.py --config 3 --calls 1 > gpurun_out/ncu_ritz.log 2>&1
echo done
