"""CPU restatement of the restarted GK mode (TEST INFRASTRUCTURE ONLY --
imported by tests/, never by the product package).

SURVEY.md 8(f) row 3: thick restart with Ritz vectors is a mode beyond the
reference's semantics (SPEC.md:155 lists restarts as a non-goal), so there is
no reference code or golden vector to pin it to; "parity unpinned" in the
reference sense.  It is checked instead against a dense SVD (converged
singular triplets are basis-independent) in tests/test_restart_oracle.py.

Same algorithm as paper_2104_10785_b200/restart.py, restated with numpy:
the GK recurrence of bidiag.py:111-178 (oracle/krylov_oracle.py) in the
transposed form A^T Q_k = P_k T, A P_k = Q_k T^T + beta_{k+1} q_{k+1} e_k^T,
restart keeping l Ritz pairs [u_1..u_l, q_{k+1}] / [v_1..v_l], resumed with
z = A^T q_{k+1} orthogonalised (CGS2) against the kept v's.
"""

from __future__ import annotations

import numpy as np

from .krylov_oracle import GK_START, _reorth, as_op, philox_stream


def restarted_oracle(A, r, k, tol=1e-10, max_restarts=100, keep=None, eps=1e-8,
                     reorth_passes=2, start_mean=2.0, start_std=1.0, seed=0):
    op = as_op(A)
    m, n = op.shape
    l_keep = min(k - 1, max(r, (k + r) // 2)) if keep is None else keep
    rng = philox_stream(seed, GK_START)
    q = start_mean + start_std * rng.standard_normal(m)
    q /= np.linalg.norm(q)
    Q = np.zeros((m, k + 1))
    P = np.zeros((n, k))
    Q[:, 0] = q
    T = np.zeros((k, k))
    l, restarts, steps = 0, 0, 0
    head = None
    while True:
        # z = A^T q_{l+1}, CGS2 against P[:, :l]
        z = op.apply_t(Q[:, l])
        z = _reorth(z, P[:, :l], reorth_passes if l else 0)
        a = float(np.linalg.norm(z))
        T[:] = 0.0
        if head is not None:
            T[:l, :l] = np.diag(head[0])
            T[:l, l] = head[1]
        kp, beta_next, alpha_break, alpha_next = k, 0.0, False, 0.0
        if a < eps:
            kp, alpha_break, alpha_next = l, True, a
        else:
            T[l, l] = a
            P[:, l] = z / a
            for i in range(l + 1, k + 1):
                w = op.apply(P[:, i - 1]) - T[i - 1, i - 1] * Q[:, i - 1]
                w = _reorth(w, Q[:, :i], reorth_passes)
                b = float(np.linalg.norm(w))
                steps += 1
                if b < eps:
                    kp, beta_next = i, b
                    break
                Q[:, i] = w / b
                if i == k:
                    beta_next = b
                    break
                z = op.apply_t(Q[:, i]) - b * P[:, i - 1]
                z = _reorth(z, P[:, :i], reorth_passes)
                a = float(np.linalg.norm(z))
                if a < eps:
                    kp, alpha_break, alpha_next = i, True, a
                    T[i - 1, i] = b
                    break
                T[i - 1, i] = b
                T[i, i] = a
                P[:, i] = z / a
        size = kp + 1 if alpha_break else kp
        Ts = T[:size, :size]
        Uh, s, Vht = np.linalg.svd(Ts)
        Vh = Vht.T
        early = kp < k or alpha_break
        # residual of each Ritz triplet: beta_{k'+1} |Uh[k'-1, i]| (A v - s u),
        # or after an alpha breakdown alpha_{k'+1} |Vh[k', i]| (A^T u - s v)
        resid = (abs(alpha_next) * np.abs(Vh[kp, :]) if alpha_break
                 else abs(beta_next) * np.abs(Uh[kp - 1, :]))
        s1 = float(s[0]) if s.size else 0.0
        take = min(r, int((s > 1e-14 * s1).sum()))
        if early or np.all(resid[:take] <= tol * s1) or restarts >= max_restarts:
            U = Q[:, :size] @ Vh[:, :take]
            V = P[:, :min(kp, size)] @ Uh[:min(kp, size), :take]
            return U, s[:take], V, restarts, resid[:take]
        l = l_keep
        Qn = np.zeros_like(Q)
        Pn = np.zeros_like(P)
        Qn[:, :l] = Q[:, :k] @ Vh[:, :l]
        Qn[:, l] = Q[:, k]
        Pn[:, :l] = P[:, :k] @ Uh[:, :l]
        head = (s[:l].copy(), beta_next * Uh[k - 1, :l])
        Q, P = Qn, Pn
        restarts += 1
