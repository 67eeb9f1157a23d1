"""Lookahead A/B helper: time GK runs of fixed length on config 2's matrix and
dump the alphas/betas (run in two processes, KSVD_LOOKAHEAD=0 / default)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import bidiag, synth

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
op = K.DeviceMatrix.from_host(synth.config2_matrix(seed=1))
out = {}
for k in (30, 60, 120):
    cfg = K.BidiagConfig(k_max=k, seed=1)
    bidiag.run_gk(op, cfg)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        run = bidiag.run_gk(op, cfg)
        ts.append(time.perf_counter() - t0)
    st = K.bidiagonalize(op, cfg)
    out[k] = {"ms_per_step": 1e3 * min(ts) / k, "alphas": list(map(float, st.alphas)),
              "betas": list(map(float, st.betas))}
print(json.dumps(out))
