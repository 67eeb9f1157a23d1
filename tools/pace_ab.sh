timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
KSVD_PHASE_TIMES=1 KSVD_DEBUG_HOST=1 timeout 300 python tools/call_breakdown.py > gpurun_out/breakdown.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
