"""CPU model of the PAIRED GK step -- TEST INFRASTRUCTURE ONLY.

Restates with numpy the arithmetic of the device's paired step
(csrc/pair.cuh, k_cgs2_pair; csrc/ksvd.cu enqueue_step; DESIGN.md 3-pair):

  w  = A p_i - alpha_i q_i                 (k_gemv_n, finalised in its tail)
  y  = A^T w                               (k_gemv_t2 on the NOT yet
                                            orthogonalised w)
  w' = CGS2(w, Q_i);  beta_{i+1} = ||w'||;  q_{i+1} = w' / beta
  y' = CGS2(y, P_i);  alpha_{i+1} = ||y'|| / beta;  p_{i+1} = y' / ||y'||

against the reference recurrence (bidiag.py:151-178), which orthogonalises w
before forming z = A^T q_{i+1} - beta p_i.  The two agree in exact
arithmetic (A^T Q_i d and beta p_i lie in span(P_i) by the GK relations);
tests/test_paired_model.py holds this model to the oracle with the parity
predicates the GPU path meets, so the reformulation itself is checked on
CPU, independently of the kernels.
"""

from __future__ import annotations

import numpy as np

from oracle.krylov_oracle import GK_START, philox_stream


def _cgs2(x, B):
    for _ in range(2):
        if B.shape[1]:
            x = x - B @ (B.T @ x)
    return x


def paired_gk(A: np.ndarray, k_max: int, eps: float = 1e-8, seed: int = 0):
    m, n = A.shape
    rng = philox_stream(seed, GK_START)
    q = 2.0 + rng.standard_normal(m)
    beta1 = float(np.linalg.norm(q))
    q /= beta1
    Q = np.zeros((m, k_max + 1))
    P = np.zeros((n, k_max))
    Q[:, 0] = q
    alphas, betas = [], [beta1]
    z = A.T @ q                              # the first product (bidiag.py:139-147)
    alpha = float(np.linalg.norm(z))
    if alpha < eps:
        return dict(alphas=np.zeros(0), betas=np.array(betas), k_prime=0, Q=Q[:, :1], P=P[:, :0])
    alphas.append(alpha)
    P[:, 0] = z / alpha
    kp = k_max
    for i in range(1, k_max + 1):
        w = A @ P[:, i - 1] - alphas[-1] * Q[:, i - 1]
        if i == k_max:                       # the last step: left side only
            w = _cgs2(w, Q[:, :i])
            beta = float(np.linalg.norm(w))
            betas.append(beta)
            if beta < eps:
                kp = i
                break
            Q[:, i] = w / beta
            break
        y = A.T @ w                          # on the raw w
        w = _cgs2(w, Q[:, :i])
        y = _cgs2(y, P[:, :i])
        beta = float(np.linalg.norm(w))
        betas.append(beta)
        if beta < eps:
            kp = i
            break
        Q[:, i] = w / beta
        ynrm = float(np.linalg.norm(y))
        alpha = ynrm / beta
        if alpha < eps:
            kp = i
            break
        alphas.append(alpha)
        P[:, i] = y / ynrm
    return dict(alphas=np.array(alphas[:kp]), betas=np.array(betas[:kp + 1]), k_prime=kp,
                Q=Q[:, :kp + 1], P=P[:, :kp])
