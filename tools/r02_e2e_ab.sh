#!/bin/bash
# upload chunk 16 MB (new default) vs 64 MB (KSVD_IO_CHUNK_BYTES=67108864): upload_bench + e2e of configs 2 and 4
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/e2e_ab; mkdir -p $O
for v in "X=1" "KSVD_IO_CHUNK_BYTES=67108864"; do echo "== $v"; env $v timeout 300 python tools/upload_bench.py 2>&1 | tail -4; done
for c in 2 4; do
for v in "X=1" "KSVD_IO_CHUNK_BYTES=67108864"; do
  env $v timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/c${c}_${v%%=*}.json 2>> $O/err.txt
  python -c "
import json; d=json.load(open('$O/c${c}_${v%%=*}.json')); print('config $c $v value', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'upload GB/s', round(d['ingest']['upload_GBps'],1), d['clocks']['sm_mhz'])"
done
done
