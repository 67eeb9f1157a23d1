#!/bin/bash
# ncu --set full of the A-streaming kernels (config 2 f64, config 4 f32)
python tools/one_call.py --config 2 --calls 1 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemv_n2|k_gemv_t<" -s 20 -c 2 -o gpurun_out/prof_c2 python tools/one_call.py --config 2 --calls 1 > gpurun_out/ncu_c2.log 2>&1
python tools/one_call.py --config 4 --calls 1 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemv_n2|k_gemv_t<" -s 20 -c 2 -o gpurun_out/prof_c4 python tools/one_call.py --config 4 --calls 1 > gpurun_out/ncu_c4.log 2>&1
