#!/bin/bash
# dram traffic per launch of the dominant kernel (ncu --set full), configs 1/3/5
mkdir -p gpurun_out
for c in ${CFGS:-1 3 5}; do
  k='regex:k_gemv_n2'
  [ $c = 1 ] && k='regex:k_gk_resident'
  python tools/one_call.py --config $c --calls 1 > gpurun_out/plain_t$c.log 2>&1 && \
  skip=3; [ $c = 1 ] && skip=0
  timeout 1500 ncu --set full --clock-control none -k "$k" -s $skip -c 1 -o gpurun_out/traffic_c$c \
    python tools/one_call.py --config $c --calls 1 > gpurun_out/ncu_t$c.log 2>&1
  ncu -i gpurun_out/traffic_c$c.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; u=rows[1]
for r in rows[2:]:
    print('config $c', r[h.index('Kernel Name')][:40], *[(k, r[h.index(k)], u[h.index(k)]) for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum']])
"
done
