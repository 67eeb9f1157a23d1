"""Compare CGS paths on a rank-exhaustion case: spurious Ritz values, orthogonality."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CODE = r"""
import sys, json
sys.path.insert(0, %r)
import numpy as np
import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth
A = synth.low_rank_synth(5000, 1200, 300, seed=9)
rep = K.estimate_rank(A, cfg=K.BidiagConfig(k_max=1, seed=9))
st = K.bidiagonalize(A, K.BidiagConfig(k_max=310, seed=9))
Q, P = st.Q, st.P
oq = float(np.max(np.abs(Q.T @ Q - np.eye(Q.shape[1]))))
op = float(np.max(np.abs(P.T @ P - np.eye(P.shape[1]))))
print(json.dumps(dict(rank=rep.rank, kp=rep.k_prime, tail=rep.eigenvalues[298:306].tolist(),
                      oq=oq, op=op, kp2=st.k_prime)))
""" % str(ROOT)
for env in ({}, {"KSVD_TILE": "0"}, {"KSVD_COOP": "0"}):
    r = subprocess.run([sys.executable, "-c", CODE], env={**os.environ, **env},
                       capture_output=True, text=True)
    print(env, r.stdout.strip() or r.stderr[-1500:])
