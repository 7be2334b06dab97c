"""Partial Cholesky preconditioner (Chol-IP-PMM, the paper's comparison arm) — ORACLE (test
infrastructure only).  SURVEY §8(f) f2.

PAPER.md:250-349 ("Partial Cholesky preconditioners"), written out:
  * N_delta = N + delta I;  diag(N_delta)_i = r_i^T r_i + delta with r_i = (Q+Theta^{-1}+rho I)^{-1/2} A^T e_i
    (P:336-340), i.e. sum_j d_j A_ij^2 + delta (+ e_i for the unit columns of the SVM operator, A23).
  * E brings the ell LARGEST diagonal entries of N_delta to the front: N_{delta,11} "is the leading
    principal submatrix containing the ell largest diagonal elements".  Reading (DESIGN.md
    C1): the pivots are the ell largest entries of the ORIGINAL diagonal (no Schur-complement
    updates of the pivot choice), ties broken by the smaller index.
  * eq.: [N11 N21^T; N21 N22] = [L11 0; L21 I] [I 0; 0 S] [L11^T L21^T; 0 I], so
    L11 = chol(N11) (lower), L21 = N21 L11^{-T}, S = N22 - N21 N11^{-1} N21^T.
  * eq. (chol-precond): P = E^T [L11 0; L21 I] [I 0; 0 diag(S)] [...]^T E.
  * eq. (chol-precond-inv): P^{-1} = E^T [L11^{-T}  -L11^{-T} L21^T; 0 I] [I 0; 0 diag(S)^{-1}]
                                                 [L11^{-1} 0; -L21 L11^{-1} I] E.
The columns N_delta[:, P] are formed matrix-free as A (d o (A^T E_P)) + delta E_P.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def diag_normal(A, d, delta, e=None):
    """diag(N + delta I) = sum_j d_j A_ij^2 (+ e_i) + delta."""
    g = (A * A) @ d
    if e is not None:
        g = g + e
    return g + delta


def pivots(diag, ell):
    """Indices of the ell largest diagonal entries (C1: original diagonal, ties -> smaller index)."""
    order = sorted(range(len(diag)), key=lambda i: (-diag[i], i))
    return np.array(order[:ell], dtype=np.int64)


def partial_cholesky(A, d, delta, ell, e=None):
    """Factors of eq.: pivots P, L11 (lower), L21 (rows of the complement, in index
    order), diag(S), and the complement indices Q."""
    m = A.shape[0]
    dg = diag_normal(A, d, delta, e)
    P = pivots(dg, ell)
    Qc = np.array([i for i in range(m) if i not in set(P.tolist())], dtype=np.int64)
    EP = np.zeros((m, ell))
    EP[P, np.arange(ell)] = 1.0
    cols = A @ (d[:, None] * (A.T @ EP)) + delta * EP              # N_delta[:, P]
    if e is not None:
        cols = cols + e[:, None] * EP
    N11 = cols[P, :]
    N21 = cols[Qc, :]
    L11 = sla.cholesky(0.5 * (N11 + N11.T), lower=True) if ell > 0 else np.zeros((0, 0))
    L21 = sla.solve_triangular(L11, N21.T, lower=True).T if ell > 0 else np.zeros((len(Qc), 0))
    dS = dg[Qc] - np.sum(L21 * L21, axis=1)                        # diag(S) = diag(N22 - L21 L21^T)
    return {"P": P, "Q": Qc, "L11": L11, "L21": L21, "dS": dS}


def chol_precond_inv_apply(F, v):
    """eq. (chol-precond-inv), applied right to left."""
    P, Qc, L11, L21, dS = F["P"], F["Q"], F["L11"], F["L21"], F["dS"]
    v1, v2 = v[P], v[Qc]                                           # E v
    u1 = sla.solve_triangular(L11, v1, lower=True) if len(P) else v1      # L11^{-1} v1
    u2 = v2 - L21 @ u1                                             # -L21 L11^{-1} v1 + v2
    w2 = u2 / dS                                                   # diag(S)^{-1}
    w1 = sla.solve_triangular(L11.T, u1 - L21.T @ w2, lower=False) if len(P) else u1   # L11^{-T}(u1 - L21^T w2)
    out = np.empty_like(v)
    out[P] = w1
    out[Qc] = w2
    return out                                                     # E^T [w1; w2]


def chol_precond_dense(F, m):
    """P_Chol as a dense matrix (eq. P:293-306) — small sizes / tests only."""
    P, Qc, L11, L21, dS = F["P"], F["Q"], F["L11"], F["L21"], F["dS"]
    ell = len(P)
    L = np.zeros((m, m))
    L[:ell, :ell] = L11
    L[ell:, :ell] = L21
    L[ell:, ell:] = np.eye(m - ell)
    Mid = np.zeros((m, m))
    Mid[:ell, :ell] = np.eye(ell)
    Mid[ell:, ell:] = np.diag(dS)
    Pp = L @ Mid @ L.T                                             # in permuted order [P; Q]
    perm = np.concatenate([P, Qc])
    Pm = np.zeros((m, m))
    Pm[np.ix_(perm, perm)] = Pp                                    # E^T (.) E
    return Pm
