timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --config 3 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
