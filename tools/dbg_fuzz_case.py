"""Debug one fuzz case: sigma / alphas of the device path vs the oracle."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
from tests.test_gpu_fuzz import _cases, _blocked

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 26
i, m, n, l, k, r, f32 = _cases()[idx]
A = synth.low_rank_synth(m, n, l, seed=1000 + i)
if f32:
    A = A.astype(np.float32)
A64 = A.astype(np.float64)
cfg = K.BidiagConfig(k_max=k, seed=i)
st = K.bidiagonalize(A, cfg)
ref = O.gk_oracle(A64, k, seed=i)
print("case", (i, m, n, l, k, r, f32), "k'", st.k_prime, ref.k_prime)
np.set_printoptions(precision=6, linewidth=200)
print("alphas dev", st.alphas[:12]); print("alphas ref", ref.alphas[:12])
print("betas dev", st.betas[:12]); print("betas ref", ref.betas[:12])
ps = K.fsvd(A, k=k, r=r, cfg=cfg)
fr = O.fsvd_oracle(A64, k, r, seed=i)
fr2 = O.fsvd_oracle(_blocked(A64), k, r, seed=i)
print("sigma dev ", ps.sigma); print("sigma ref ", fr.sigma); print("sigma ref2", fr2.sigma)
nt = min(ps.sigma.size, fr.sigma.size, fr2.sigma.size)
spread = np.abs(fr.sigma[:nt] - fr2.sigma[:nt])
print("dev-ref rel ", np.abs(ps.sigma[:nt] - fr.sigma[:nt]) / fr.sigma[:nt])
print("spread rel  ", spread / fr.sigma[:nt])
th = np.sort(np.abs(np.linalg.svd(np.diag(st.alphas) + np.diag(st.betas[1:len(st.alphas)], -1)[:len(st.alphas), :len(st.alphas)], compute_uv=False)))[::-1]
print("alphas rel diff (all)", np.max(np.abs(st.alphas - ref.alphas) / np.abs(ref.alphas)))
