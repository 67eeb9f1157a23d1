#!/bin/bash
python tools/one_call.py --config 4 --calls 1 > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/one_call.py --config 4 --calls 1 > gpurun_out/ncu_c4.log 2>&1
python tools/one_call.py --config 5 --calls 1 > gpurun_out/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/one_call.py --config 5 --calls 1 > gpurun_out/ncu_c5.log 2>&1
