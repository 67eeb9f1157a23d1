#!/bin/bash
# round-2 re-entry validation: box facts, the whole GPU suite (slow full-size
# tests included), then every config through bench.py (both arms)
cd "${GRAFT_REPO_ROOT:-.}"
O=${VAL_OUT:-gpurun_out/r02b}; mkdir -p $O
(nvidia-smi; free -g; nproc; lscpu | head -20) > $O/box.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=15 > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
tail -25 $O/gpu_tests.log
bash tools/bench_all_r02.sh
