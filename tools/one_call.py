"""Run the bench workload once after a warm-up (target for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import argparse

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--calls", type=int, default=2)
a = ap.parse_args()
if a.config == 2:
    A = synth.config2_matrix(seed=1)
    op = K.DeviceMatrix.from_host(A)
    for _ in range(a.calls):
        rep = K.estimate_rank(op, eps=1e-6, mode="relative", cfg=K.BidiagConfig(k_max=1, seed=1))
    print("rank", rep.rank, "k'", rep.k_prime)
else:
    A = synth.config1_matrix(seed=0)
    op = K.DeviceMatrix.from_host(A)
    for _ in range(a.calls):
        ps = K.fsvd(op, k=30, r=10, cfg=K.BidiagConfig(k_max=30, eps=1e-10, seed=0))
    print("sigma", ps.sigma[:3])
