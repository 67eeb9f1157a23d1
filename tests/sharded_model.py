"""CPU model of the row-sharded GK loop -- TEST INFRASTRUCTURE ONLY.

Restates, rank by rank with numpy, exactly the data movement the CUDA path
performs at N GPUs (csrc/ksvd.cu: enqueue_step / cgs_impl / enqueue_gemv_t):

  left  (row-sharded q, Q): w_loc = A_loc p - alpha q_loc (local);
        c = allreduce(Q_loc^T w_loc); w_loc -= Q_loc c   (twice for CGS2);
        beta^2 = allreduce(|w_loc|^2) (+ the non-finite flag)
  right (replicated p, P):  z = allreduce(A_loc^T q_loc) - beta p;
        CGS2 and alpha computed redundantly on every rank (no collective)

The collectives go through torch.distributed (gloo here; NCCL on the GPU
box), so a world_size-2 run on CPU checks the partitioning and the
collective arithmetic against the single-process oracle.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from oracle.krylov_oracle import GK_START, philox_stream
from paper_2104_10785_b200.linops import row_partition


def allreduce(x: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64).copy())
    dist.all_reduce(t)
    return t.numpy()


def sharded_gk(A_full: np.ndarray, k_max: int, eps: float = 1e-8, seed: int = 0,
               passes: int = 2):
    rank, world = dist.get_rank(), dist.get_world_size()
    m, n = A_full.shape
    r0, ml = row_partition(m, world, rank)
    A = A_full[r0:r0 + ml]
    rng = philox_stream(seed, GK_START)
    q = 2.0 + rng.standard_normal(m)
    beta1 = float(np.linalg.norm(q))
    q /= beta1
    Q = np.zeros((ml, k_max + 1))
    P = np.zeros((n, k_max))
    Q[:, 0] = q[r0:r0 + ml]
    alphas, betas = [], [beta1]

    z = allreduce(A.T @ Q[:, 0])
    alpha = float(np.sqrt(z @ z))
    if alpha < eps:
        return dict(alphas=np.zeros(0), betas=np.array(betas), k_prime=0, Q=Q[:, :1], P=P[:, :0])
    alphas.append(alpha)
    kp, why = k_max, ""
    for i in range(1, k_max + 1):
        P[:, i - 1] = z / alphas[-1]
        w = A @ P[:, i - 1] - alphas[-1] * Q[:, i - 1]
        for _ in range(passes):
            c = allreduce(Q[:, :i].T @ w)
            w = w - Q[:, :i] @ c
        red = allreduce(np.array([w @ w, float(not np.isfinite(w).all())]))
        if red[1]:
            raise FloatingPointError("non-finite")
        beta = float(np.sqrt(red[0]))
        betas.append(beta)
        if beta < eps:
            kp, why = i, "beta"
            break
        Q[:, i] = w / beta
        if i == k_max:
            break
        z = allreduce(A.T @ Q[:, i]) - beta * P[:, i - 1]
        for _ in range(passes):
            z = z - P[:, :i] @ (P[:, :i].T @ z)
        alpha = float(np.sqrt(z @ z))
        if alpha < eps:
            kp, why = i, "alpha"
            break
        alphas.append(alpha)
    return dict(alphas=np.array(alphas), betas=np.array(betas), k_prime=kp, breakdown=why,
                Q=Q[:, :kp + 1], P=P[:, :kp], row0=r0)
