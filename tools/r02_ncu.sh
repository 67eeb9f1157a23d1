#!/bin/bash
# round-2 ncu evidence: launch lists (config 2, config 4) and --set full of
# the top kernels (k_gemv_n / k_gemv_t2 on config 4, k_cgs2_tile2 on config 2)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ncu2; mkdir -p $O
python tools/one_call.py --config 2 --calls 1 > $O/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches_c2.csv \
    python tools/one_call.py --config 2 --calls 1 > $O/ncu_list_c2.log 2>&1
python tools/one_call.py --config 2 --calls 1 > $O/plain_c2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_cgs2_tile2" -s 160 -c 3 \
    -o $O/prof_cgs_c2 python tools/one_call.py --config 2 --calls 1 > $O/ncu_cgs_c2.log 2>&1
python tools/one_call.py --config 4 --calls 1 > $O/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches_c4.csv \
    python tools/one_call.py --config 4 --calls 1 > $O/ncu_list_c4.log 2>&1
python tools/one_call.py --config 4 --calls 1 > $O/plain_c4b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemv_n<|k_gemv_t2" -s 40 -c 2 \
    -o $O/prof_gemv_c4 python tools/one_call.py --config 4 --calls 1 > $O/ncu_gemv_c4.log 2>&1
ls -la $O
