#!/bin/bash
# round-2 final ncu evidence (each command first runs clean without ncu):
# launch lists of one call (configs 2, 4), DRAM bytes per launch of the two
# A-streaming kernels (configs 2-5), a full capture of k_cgs2_pair (config 2)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ncu_final; mkdir -p $O
for c in 2 4; do
  python tools/one_call.py --config $c --calls 1 > $O/plain_c$c.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c$c.csv \
      python tools/one_call.py --config $c --calls 1 > $O/ncu_list_c$c.log 2>&1
  python tools/launch_summary.py $O/launches_c$c.csv > $O/launches_config$c.txt
  cat $O/launches_config$c.txt
done
for c in 2 3 4 5; do
  timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"k_gemv_n|k_gemv_t2" -s 20 -c 4 --csv --log-file $O/traffic_c$c.csv \
      python tools/one_call.py --config $c --calls 1 > $O/ncu_traffic_c$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cgs2_pair" -s 120 -c 2 \
    -o $O/prof_pair_c2 python tools/one_call.py --config 2 --calls 1 > $O/ncu_pair_c2.log 2>&1
ls -la $O
