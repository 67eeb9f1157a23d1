"""Input recipes of the golden cases (no reference import needed)."""

from __future__ import annotations

import hashlib

import numpy as np

from paper_2104_10785_b200 import synth


def digest(A) -> str:
    return hashlib.sha256(np.ascontiguousarray(A, dtype=np.float64).tobytes()).hexdigest()[:16]


# Input recipes (also used by the tests to rebuild the inputs).
def build_input(recipe: str) -> np.ndarray:
    kind, *args = recipe.split(":")
    a = [float(x) if "." in x or "e" in x else int(x) for x in args]
    if kind == "lowrank":
        return synth.low_rank_synth(*a[:3], seed=a[3])
    if kind == "gauss":
        return synth.gaussian_matrix(a[0], a[1], seed=a[2])
    if kind == "eye":
        return np.eye(a[0])
    if kind == "zeros":
        return np.zeros((a[0], a[1]))
    if kind == "diag":
        return np.diag(np.array(a, dtype=np.float64))
    if kind == "paddiag":  # zeros(m, n) with diag(vals) in the corner
        m, n, *vals = a
        A = np.zeros((m, n))
        A[:len(vals), :len(vals)] = np.diag(np.array(vals, dtype=np.float64))
        return A
    if kind == "config1":
        return synth.config1_matrix(seed=0)
    raise ValueError(recipe)


