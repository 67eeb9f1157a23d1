#!/bin/bash
# full GPU test suite + smoke + bench lines for configs 1-5 + resident-kernel ncu
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log
bash tools/bench_all.sh
python tools/one_call.py --config 1 --calls 1 > gpurun_out/plain_r.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gk_resident -c 1 \
  -o gpurun_out/prof_resident python tools/one_call.py --config 1 --calls 1 > gpurun_out/ncu_resident.log 2>&1
echo done
