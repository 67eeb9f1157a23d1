#!/bin/bash
# cluster CGS2: parity of every path, then config-2 A/B of the cluster sizes
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02c; mkdir -p $O
KSVD_DEBUG_HOST=1 python -c "import sys; sys.path.insert(0,'.'); from paper_2104_10785_b200 import _lib; _lib.get_context()" > $O/probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "paths_agree or golden" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
for i in 1 2; do
  for cs in 1 2 4 8; do
    KSVD_CGS_CLUSTER=$cs timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/c2_cs${cs}_$i.json 2>> $O/ab.err
  done
  timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/c2_def_$i.json 2>> $O/ab.err
done
KSVD_PHASE_TIMES=1 KSVD_CGS_CLUSTER=1 timeout 300 python tools/one_call.py --config 2 > $O/phases_cs1.txt 2>&1
KSVD_PHASE_TIMES=1 timeout 300 python tools/one_call.py --config 2 > $O/phases_def.txt 2>&1
for f in $O/c2_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read()); print(round(d['value'],1), round(d['roofline']['share_of_device_time']['cgs'],4))")"; done
cat $O/probe.txt; tail -2 $O/parity.log
