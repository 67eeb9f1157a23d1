#!/bin/bash
# ncu --set full of the final k_gemv_n (named barriers, evict_first) and k_gemv_t2 on config 4
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ncu_c4; mkdir -p $O
python tools/one_call.py --config 4 --calls 1 > $O/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"^k_gemv_n$" -s 10 -c 1 \
    -o $O/prof_gemvn_c4 python tools/one_call.py --config 4 --calls 1 > $O/ncu.log 2>&1
ls -la $O
