"""Normal-equation operator of IP-PMM — ORACLE (test infrastructure only).

PAPER.md:197-205 (eq. normal-eq): (N_k + delta_k I) dy = xi, with
    N_k = A (Q + Theta_k^{-1} + rho_k I)^{-1} A^T,   Theta_k = diag(x) diag(z)^{-1}.
We write D = (Q + Theta^{-1} + rho I)^{-1} = diag(d).  PAPER.md:755 builds N_k "as a linear
operator"; P:835 solves with [A D A^T + delta I].  The optional diagonal `e` is the
contribution of unit columns of A (the SVM config's xi/s columns), so that
    w = A (d o (A^T v)) + e o v + delta v.
"""
from __future__ import annotations

import numpy as np


def scaling_d(q, x, z, rho):
    """d_j = 1 / (q_j + z_j / x_j + rho)   (P:201 with Theta^{-1} = diag(z/x))."""
    return 1.0 / (q + z / x + rho)


def normal_matvec(A, d, v, delta, e=None):
    """w = A diag(d) A^T v + e o v + delta v, evaluated in that order."""
    t = d * (A.T @ v)
    w = A @ t
    if e is not None:
        w = w + e * v
    return w + delta * v


def sketch(A, d, Omega, e=None):
    """Y = N Omega with N = A diag(d) A^T (+ diag(e)), WITHOUT delta (Alg. 1 line 2)."""
    T = d[:, None] * (A.T @ Omega)
    Y = A @ T
    if e is not None:
        Y = Y + e[:, None] * Omega
    return Y


def dense_normal_matrix(A, d, delta, e=None):
    """Materialised N + delta I (path D of the oracle and small-size tests only)."""
    N = (A * d[None, :]) @ A.T
    if e is not None:
        N = N + np.diag(e)
    return N + delta * np.eye(A.shape[0])
