"""Seeded synthetic inputs.

`gaussian_matrix` / `low_rank_synth` keep the reference generators' streams
(linops.py:217-240) so the reference's test matrices are reproduced bit for
bit.  `baseline_config(i)` builds the BASELINE.json configurations that fit
host memory (configs 1-2) on the host with numpy; configs 3-5 are too large
for a host oracle and are generated on the device.
No public dataset is involved: everything is synthetic.
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigError
from .linops import substream

GAUSS, SYNTH_LEFT, SYNTH_RIGHT, BENCH_MATRIX = 1, 2, 3, 12  # reference tags


def gaussian_matrix(m: int, n: int, mean: float = 0.0, std: float = 1.0,
                    seed: int = 0) -> np.ndarray:
    if m < 1 or n < 1:
        raise ConfigError(f"matrix dims must be >= 1, got {m}x{n}")
    if not std > 0:
        raise ConfigError(f"std must be > 0, got {std}")
    return mean + std * substream(seed, GAUSS).standard_normal((m, n))


def low_rank_synth(m: int, n: int, l: int, seed: int = 0) -> np.ndarray:
    if m < 1 or n < 1:
        raise ConfigError(f"matrix dims must be >= 1, got {m}x{n}")
    if not 1 <= l <= min(m, n):
        raise ConfigError(f"rank l must be in [1, min(m,n)]; got l={l} for {m}x{n}")
    return (substream(seed, SYNTH_LEFT).standard_normal((m, l))
            @ substream(seed, SYNTH_RIGHT).standard_normal((l, n)))


def config1_matrix(seed: int = 0, m: int = 2000, n: int = 1000) -> np.ndarray:
    """BASELINE config 1: A = U diag(s) V^T, U/V = Q factors of QR of iid
    N(0,1), s_i = 10^(-4(i-1)/(n-1)) geometric from 1 to 1e-4."""
    rng = substream(seed, BENCH_MATRIX)
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = 10.0 ** (-4.0 * np.arange(n) / (n - 1))
    return (U * s) @ V.T


def config2_matrix(seed: int = 1, m: int = 20000, n: int = 5000, r: int = 137,
                   noise: float = 1e-10, dtype=np.float64, out=None) -> np.ndarray:
    """BASELINE config 2: A = X Y^T + E, X/Y iid N(0, 1/r), E iid N(0, noise^2).
    `out` may be a preallocated (e.g. pinned) m x n float64 array."""
    rng = substream(seed, BENCH_MATRIX)
    X = rng.standard_normal((m, r)) / np.sqrt(r)
    Y = rng.standard_normal((n, r)) / np.sqrt(r)
    A = out if out is not None else np.empty((m, n), dtype=np.float64)
    step = 2048
    for i0 in range(0, m, step):  # bounded temporaries
        i1 = min(m, i0 + step)
        A[i0:i1] = X[i0:i1] @ Y.T + noise * rng.standard_normal((i1 - i0, n))
    return A.astype(dtype, copy=False)


# (call, kwargs) of each BASELINE.json config that the host can build
BASELINE_CALLS = {
    1: dict(kind="fsvd", k=30, r=10, eps=1e-10, seed=0),
    2: dict(kind="rank", eps=1e-6, mode="relative", seed=1),
}
