#!/bin/bash
# ncu launch list of one config-2 call with the paired step + a full capture
# of k_cgs2_pair (late steps)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ncu_pair; mkdir -p $O
python tools/one_call.py --config 2 --calls 1 > $O/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches_c2.csv \
    python tools/one_call.py --config 2 --calls 1 > $O/ncu_list_c2.log 2>&1
python tools/launch_summary.py $O/launches_c2.csv > $O/launches_config2.txt
cat $O/launches_config2.txt
ncu --set full --clock-control none --import-source on -k regex:"k_cgs2_pair" -s 120 -c 2 \
    -o $O/prof_pair_c2 python tools/one_call.py --config 2 --calls 1 > $O/ncu_pair_c2.log 2>&1
ls -la $O
