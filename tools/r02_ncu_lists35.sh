#!/bin/bash
# final-build ncu launch lists of one call, configs 3 and 5 (each first run clean)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ncu_final35; mkdir -p $O
for c in 3 5; do
  python tools/one_call.py --config $c --calls 1 > $O/plain_c$c.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c$c.csv \
      python tools/one_call.py --config $c --calls 1 > $O/ncu_list_c$c.log 2>&1
  python tools/launch_summary.py $O/launches_c$c.csv > $O/launches_config$c.txt
  head -12 $O/launches_config$c.txt
done
