#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/la_dbg3; mkdir -p $O
cat > /tmp/dbg.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import bidiag, synth
ks = [int(x) for x in sys.argv[1:]]
op = K.DeviceMatrix.from_host(synth.config2_matrix(seed=1))
for k in ks:
    try:
        st = K.bidiagonalize(op, K.BidiagConfig(k_max=k, seed=1))
        print(k, "ok", st.alphas[-3:], st.betas[-3:], flush=True)
    except Exception as e:
        print(k, "ERR", e, flush=True)
rep = K.estimate_rank(op, eps=1e-6, mode="relative", cfg=K.BidiagConfig(k_max=1, seed=1))
print("rank", rep.rank, rep.k_prime, flush=True)
PY
for env in "KSVD_LOOKAHEAD=0" "KSVD_PDL=0" "X=1"; do
  echo "== $env" >> $O/out.txt
  env $env KSVD_DEBUG_STATE=1 timeout 120 python /tmp/dbg.py 4 8 30 60 120 >> $O/out.txt 2>&1
done
cat $O/out.txt
bash tools/r02_la_t.sh
