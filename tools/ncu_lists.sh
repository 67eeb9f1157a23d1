#!/bin/bash
# ncu launch lists (gpu__time_duration.sum, cold-cache serialised) of one call, configs 4 and 5
for c in ${CFGS:-4 5}; do
python tools/one_call.py --config $c --calls 1 > gpurun_out/plain_c$c.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv python tools/one_call.py --config $c --calls 1 > gpurun_out/ncu_c$c.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c$c.csv > gpurun_out/launches_config$c.txt
done
