import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth, _lib
from paper_2104_10785_b200.bidiag import run_gk
from paper_2104_10785_b200.restart import _info, _projected
A = synth.low_rank_synth(500, 300, 6, seed=2)
run = run_gk(K.DeviceMatrix.from_host(A), K.BidiagConfig(k_max=12, seed=3))
kp, flags, a, b = _info(run.handle, 12)
np.set_printoptions(linewidth=200, precision=4)
print("kp", kp, "flags", flags, "run.kp", run.k_prime)
print("a", a)
print("b", b)
T, kq, kpc = _projected(a, b, kp, flags)
print(T)
