"""Host-side launch cost probe (torch tiny kernels) + CPU info."""
import os
import time

import torch

print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
print(open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0])
x = torch.zeros(1024, device="cuda")
for _ in range(100):
    x.add_(1)
torch.cuda.synchronize()
for n in (1000, 10000):
    t0 = time.perf_counter()
    for _ in range(n):
        x.add_(1)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{n} launches: enqueue {1e6 * (t1 - t0) / n:.2f} us/launch, total {1e6 * (t2 - t0) / n:.2f} us/launch")
print(os.popen("uptime").read())
print(os.popen("nproc; cat /sys/fs/cgroup/cpu.max 2>/dev/null").read())
