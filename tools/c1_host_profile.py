"""Host-side profile of config 1's fsvd call (cProfile over repeated calls)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth

op = K.DeviceMatrix.from_host(synth.config1_matrix(seed=0))
cfg = K.BidiagConfig(k_max=30, eps=1e-10, seed=0)
for _ in range(20):
    K.fsvd(op, k=30, r=10, cfg=cfg)
t0 = time.perf_counter()
for _ in range(200):
    K.fsvd(op, k=30, r=10, cfg=cfg)
print(f"per call {1e3 * (time.perf_counter() - t0) / 200:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    K.fsvd(op, k=30, r=10, cfg=cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
