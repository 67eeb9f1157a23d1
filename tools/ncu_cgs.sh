#!/bin/bash
# ncu --set full (with source) of late-step k_cgs2_tile2 launches on config 2
mkdir -p gpurun_out
python tools/one_call.py --config 2 --calls 1 > gpurun_out/plain_c2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_cgs2_tile2" -s 200 -c 2 -o gpurun_out/prof_cgs_c2 -f \
  python tools/one_call.py --config 2 --calls 1 > gpurun_out/ncu_cgs_c2.log 2>&1
echo done
