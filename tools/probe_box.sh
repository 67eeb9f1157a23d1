set -x
free -g; nproc; lscpu | head -20; nvidia-smi; df -h /tmp /dev/shm; ulimit -l
python -c "import os; print(os.sched_getaffinity(0).__len__())"
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15
