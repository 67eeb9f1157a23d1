"""Generate golden vectors from the REFERENCE implementation (krysvd).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs tests/golden/golden.npz (small: every case fits in a few MB).  The
inputs are regenerated at test time from the same seeded generators
(paper_2104_10785_b200.synth mirrors the reference's streams bit for bit, and
each case stores a checksum of its input so a drifted generator fails
loudly).  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

import krysvd  # noqa: E402  (the reference, from PYTHONPATH)
from krysvd import (BidiagConfig, bidiagonalize, estimate_rank, fsvd,  # noqa: E402
                    gaussian_matrix, low_rank_synth, symtridiag_eig, SymTridiag)
from krysvd.linops import GK_START, substream  # noqa: E402

from paper_2104_10785_b200 import synth  # noqa: E402
from tests.golden.recipes import build_input, digest  # noqa: E402


BIDIAG_CASES = [
    # recipe, k_max, seed, reorth
    ("lowrank:60:40:20:21", 40, 21, 2),
    ("lowrank:40:60:15:19", 40, 19, 2),
    ("lowrank:128:96:40:60", 96, 60, 2),
    ("lowrank:200:150:40:80", 150, 80, 2),
    ("lowrank:40:30:10:23", 30, 23, 1),
    ("lowrank:80:60:20:31", 40, 31, 2),
    ("eye:5", 5, 7, 2),
    ("zeros:6:4", 4, 3, 2),
    ("paddiag:8:6:4:3:2:1", 6, 11, 2),
    ("gauss:30:30:13", 30, 13, 2),
    ("gauss:50:30:17", 30, 17, 2),
    ("gauss:8:8:1", 4, 42, 2),
    ("lowrank:1000:1000:100:5", 300, 5, 2),
]

FSVD_CASES = [
    # recipe, k, r, seed, eps, orthonormalize_u
    ("diag:3.0:2.0:1.0", 3, 3, 0, 1e-8, True),
    ("lowrank:200:150:40:6", 60, 40, 6, 1e-8, True),
    ("gauss:120:90:8", 90, 10, 8, 1e-8, True),
    ("lowrank:30:30:5:9", 30, 10, 0, 1e-8, True),
    ("lowrank:80:60:15:12", 40, 15, 12, 1e-8, False),
    ("lowrank:60:50:12:10", 30, 12, 10, 1e-8, True),
    ("zeros:6:4", 4, 2, 0, 1e-8, True),
    ("lowrank:100:80:40:3", 20, 20, 3, 1e-8, True),
    ("lowrank:1000:1000:100:5", 1000, 1000, 0, 1e-8, True),
    ("config1", 30, 10, 0, 1e-10, True),
]

RANK_CASES = [
    # recipe, eps, mode, seed
    ("paddiag:6:4:5.0:3.0", 1e-8, "absolute", 0),
    ("zeros:5:3", 1e-8, "absolute", 0),
    ("lowrank:1000:1000:100:7", 1e-8, "absolute", 7),
    ("lowrank:1000:1000:100:0", 1e-8, "absolute", 0),
    ("lowrank:50:40:10:8", 1e-6, "relative", 0),
    ("eye:5", 1e-8, "absolute", 0),
    ("lowrank:60:60:12:9", 1e-8, "absolute", 0),
    ("lowrank:60:60:12:9", 1e-12, "absolute", 0),
    ("lowrank:60:60:12:9", 1e-2, "absolute", 0),
    ("lowrank:80:70:20:11", 1e-8, "absolute", 11),
]


def main():
    # our generators must reproduce the reference's streams bit for bit
    assert np.array_equal(synth.low_rank_synth(60, 40, 20, seed=21),
                          low_rank_synth(60, 40, 20, seed=21))
    assert np.array_equal(synth.gaussian_matrix(30, 30, seed=13),
                          gaussian_matrix(30, 30, seed=13))
    out: dict[str, np.ndarray] = {}
    meta = []
    # start-vector stream pins (test_bidiag.py:57-75)
    for seed, m, mean, std in [(42, 8, 2.0, 1.0), (9, 6, -1.0, 0.5), (0, 2000, 2.0, 1.0)]:
        q = mean + std * substream(seed, GK_START).standard_normal(m)
        q /= np.linalg.norm(q)
        out[f"start/{seed}/{m}/{mean}/{std}"] = q
    for idx, (recipe, k, seed, reorth) in enumerate(BIDIAG_CASES):
        A = build_input(recipe)
        st = bidiagonalize(A, BidiagConfig(k_max=k, seed=seed, reorth_passes=reorth))
        p = f"bidiag/{idx}"
        out[p + "/alphas"] = st.alphas
        out[p + "/betas"] = st.betas
        out[p + "/info"] = np.array([st.k_prime, st.terminated_early, st.degenerate,
                                     st.Q.shape[1], st.P.shape[1]])
        if A.size <= 40000:
            out[p + "/Q"] = st.Q
            out[p + "/P"] = st.P
        meta.append(f"{p}|{recipe}|{k}|{seed}|{reorth}|{digest(A)}")
    for idx, (recipe, k, r, seed, eps, ortho) in enumerate(FSVD_CASES):
        A = build_input(recipe)
        psvd, st, theta = fsvd(A, k=k, r=r, cfg=BidiagConfig(k_max=k, seed=seed, eps=eps),
                               orthonormalize_u=ortho, return_details=True)
        p = f"fsvd/{idx}"
        out[p + "/sigma"] = psvd.sigma
        out[p + "/theta"] = theta
        out[p + "/info"] = np.array([psvd.truncated, psvd.n_dropped, st.k_prime,
                                     psvd.sigma.shape[0]])
        keep = min(psvd.sigma.shape[0], 40)
        out[p + "/U"] = psvd.U[:, :keep]
        out[p + "/V"] = psvd.V[:, :keep]
        meta.append(f"{p}|{recipe}|{k}|{r}|{seed}|{eps}|{int(ortho)}|{digest(A)}")
    for idx, (recipe, eps, mode, seed) in enumerate(RANK_CASES):
        A = build_input(recipe)
        rep = estimate_rank(A, eps=eps, mode=mode, cfg=BidiagConfig(k_max=1, seed=seed))
        p = f"rank/{idx}"
        out[p + "/info"] = np.array([rep.rank, rep.k_prime])
        out[p + "/eigenvalues"] = rep.eigenvalues
        out[p + "/threshold"] = np.array([rep.threshold])
        meta.append(f"{p}|{recipe}|{eps}|{mode}|{seed}|{digest(A)}")
    # eigen-solver known answers (fsvd.py:63-134 via the reference)
    for n in [1, 2, 3, 5, 13, 50, 120]:
        rng = np.random.default_rng(100 + n)
        d = rng.standard_normal(n) * 3.0
        e = rng.standard_normal(max(n - 1, 0))
        theta, G = symtridiag_eig(SymTridiag(d, e))
        out[f"eig/{n}/d"], out[f"eig/{n}/e"] = d, e
        out[f"eig/{n}/theta"], out[f"eig/{n}/G"] = theta, G
    out["meta"] = np.array(meta)
    out["reference_version"] = np.array([krysvd.__version__])
    np.savez_compressed(HERE / "golden.npz", **out)
    print(f"wrote {HERE / 'golden.npz'} ({(HERE / 'golden.npz').stat().st_size / 1e6:.2f} MB),"
          f" {len(meta)} cases")


if __name__ == "__main__":
    main()
