"""Randomized Nystrom approximation and preconditioner — ORACLE (test infrastructure only).

Alg. 1 ("Randomized Nystrom Approximation"), written line by line:
    1  Omega ~ N(0,1)^{m x l}                 (passed in: SURVEY A6)
    2  Y = N Omega                            (passed in / oracle.linops.sketch)
    3  nu = eps(norm(Y, 'fro'))               (A2: Julia eps(x) = ulp spacing at x = np.spacing)
    4  Y_nu = Y + nu Omega
    5  C = chol(Omega^T Y_nu)                 (A3: symmetrise first; C upper, C^T C = G)
    6  B = Y_nu C^{-1}
    7  [U, Sigma, ~] = svd(B)                 (thin SVD, LAPACK via numpy)
    8  Lambda = max{0, Sigma^2 - nu I}
A4 (paper silent): if the Cholesky fails, nu <- 10 nu and retry, at most 3 retries.

Eq., Alg. 2:
    P     = 1/(lam_l + mu) U (Lam + mu I) U^T + (I - U U^T)
    P^{-1} = (lam_l + mu) U (Lam + mu I)^{-1} U^T + (I - U U^T)
with mu = delta_k.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


class CholeskyFailure(RuntimeError):
    pass


def nystrom_from_sketch(Y, Omega, max_retries: int = 3):
    """Alg. 1 lines 3-8 given Y = N Omega.  Returns (U, lam, info)."""
    nu = float(np.spacing(np.linalg.norm(Y, "fro")))             # line 3
    retries = 0
    while True:
        Ynu = Y + nu * Omega                                     # line 4
        G = Omega.T @ Ynu
        G = 0.5 * (G + G.T)                                      # A3
        try:
            C = np.linalg.cholesky(G).T                          # line 5 (upper, C^T C = G)
            break
        except np.linalg.LinAlgError:
            if retries >= max_retries:
                raise CholeskyFailure("Omega^T Y_nu not positive definite after retries")
            retries += 1
            nu *= 10.0                                           # A4
    # line 6: B = Y_nu C^{-1}  <=>  C^T B^T = Y_nu^T
    B = sla.solve_triangular(C, Ynu.T, trans="T", lower=False).T
    U, S, _ = np.linalg.svd(B, full_matrices=False)              # line 7
    lam = np.maximum(0.0, S * S - nu)                            # line 8
    return U, lam, {"nu": nu, "retries": retries}


def nystrom_approx(apply_N_block, m: int, ell: int, Omega):
    """Full Alg. 1 with the sketch computed from a block operator apply_N_block(Omega) = N Omega."""
    Y = apply_N_block(Omega)                                     # line 2
    return nystrom_from_sketch(Y, Omega)


def precond_inv_apply(U, lam, mu, v):
    """P^{-1} v = (lam_l + mu) U (Lam + mu I)^{-1} U^T v + v - U U^T v."""
    g = U.T @ v
    lam_l = lam[-1]
    return (lam_l + mu) * (U @ (g / (lam + mu))) + v - U @ g


def precond_apply(U, lam, mu, v):
    """P v = 1/(lam_l + mu) U (Lam + mu I) U^T v + v - U U^T v."""
    g = U.T @ v
    lam_l = lam[-1]
    return (U @ ((lam + mu) * g)) / (lam_l + mu) + v - U @ g


def precond_inv_dense(U, lam, mu):
    m = U.shape[0]
    lam_l = lam[-1]
    return (lam_l + mu) * (U * (1.0 / (lam + mu))[None, :]) @ U.T + np.eye(m) - U @ U.T


def precond_apply_flops(m: int, ell: int) -> int:
    """Table 2 matvec cost of P^{-1}: 2 l m + m + 5 l."""
    return 2 * ell * m + m + 5 * ell
