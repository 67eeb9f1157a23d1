"""Run one BASELINE config's entry point `--calls` times (target for ncu)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--calls", type=int, default=2)
a = ap.parse_args()
call = synth.BASELINE_CALLS[a.config]
if a.config == 1:
    op = K.DeviceMatrix.from_host(synth.config1_matrix(seed=0))
elif a.config == 2:
    op = K.DeviceMatrix.from_host(synth.config2_matrix(seed=1))
else:
    op = synth.generate(synth.BASELINE_SPECS[a.config])
for _ in range(a.calls):
    if call["kind"] == "fsvd":
        out = K.fsvd(op, k=call["k"], r=call["r"],
                     cfg=K.BidiagConfig(k_max=call["k"], eps=call["eps"], seed=call["seed"]))
        msg = f"sigma[:3] {out.sigma[:3]}"
    else:
        out = K.estimate_rank(op, eps=call["eps"], mode=call["mode"],
                              cfg=K.BidiagConfig(k_max=1, seed=call["seed"]))
        msg = f"rank {out.rank} k' {out.k_prime}"
print(f"config {a.config}: {msg}")
