#!/bin/bash
# config-2 bench through the multi-rank code path on one GPU (1-rank
# communicator): NCCL all-reduces vs the NVLink peer-exchange kernels
for e in KSVD_NONE=1 KSVD_FORCE_NCCL=1 "KSVD_FORCE_NCCL=1 KSVD_PDL_MULTI=0" KSVD_FORCE_PX=1 "KSVD_FORCE_PX=1 KSVD_PDL_MULTI=0" KSVD_FORCE_NCCL=1 "KSVD_FORCE_NCCL=1 KSVD_PDL_MULTI=0"; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mu.json 2>> gpurun_out/mu_err.log
  python -c "
import json;d=json.load(open('gpurun_out/mu.json'));print('$e', round(d['value'],1), round(d['ms_per_step'],3), d['gpu_launches'], {k: round(v,3) for k,v in d['roofline']['share_of_device_time'].items()})"
done
