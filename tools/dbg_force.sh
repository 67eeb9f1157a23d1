#!/bin/bash
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d1.json 2> gpurun_out/d1.err; echo "rc1=$?"
env KSVD_FORCE_NCCL=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d2.json 2> gpurun_out/d2.err; echo "rc2=$?"
KSVD_FORCE_NCCL=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d3.json 2> gpurun_out/d3.err; echo "rc3=$?"
ls -la gpurun_out/d*
