#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/fuzz; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_restart.py tests/test_gpu_acceptance.py -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -8 $O/tests.log
