python -c "
import ctypes
cudart = ctypes.CDLL('libcudart.so.12') if False else None
" ; for v in 1 0; do KSVD_L2_PERSIST=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_l2_$v.log 2>&1; done
nvidia-smi -q | grep -i -A2 "l2\|persist" | head -20 > gpurun_out/smi_l2.txt
