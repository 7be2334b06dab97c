"""The SVM-shaped constraint operator of BASELINE config 2 and its exact Woodbury direct solve —
ORACLE (test infrastructure only).  SURVEY §8(c) "Path D ... For config 2, use the exact
Woodbury/capacitance form"; reading A23.

Config 2's QP (BASELINE.json configs[2]; the primal soft-margin SVM, App. C.2,
P:1522-1553) has variables [w+, w-, xi, s] >= 0 (sizes d, d, N, N) and constraints
    diag(y) X (w+ - w-) + xi - s = 1,
so A = [Xt, -Xt, I, -I] with Xt = diag(y) X (N x d).  A is never materialised (40.8 GB at full
size): this class applies it and its transpose.  For a scaling D = diag(d) split as
(d_w+, d_w-, d_xi, d_s), the normal matrix of P:201 is
    N + delta I = A D A^T + delta I = Xt W Xt^T + E,   W = diag(d_w+ + d_w-),  E = diag(d_xi + d_s + delta)
(the -Xt block contributes Xt D_w- Xt^T with the same sign; each unit column contributes its d_j
on the diagonal).  Its inverse is the Sherman-Morrison-Woodbury identity (textbook; Golub & Van
Loan §2.1.4) with the d x d capacitance matrix C = W^{-1} + Xt^T E^{-1} Xt:
    (N + delta I)^{-1} r = E^{-1} r - E^{-1} Xt C^{-1} Xt^T E^{-1} r,
an exact direct solve in O(N d^2) instead of the O(N^3) dense Cholesky.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


class _Transposed:
    def __init__(self, op):
        self.op = op
        self.shape = (op.shape[1], op.shape[0])

    def __matmul__(self, v):
        return self.op.rmatmul(v)

    @property
    def T(self):
        return self.op


class SvmOperator:
    """A = [Xt, -Xt, I, -I] (N x (2d + 2N)) applied without materialising it."""

    def __init__(self, Xt):
        self.Xt = np.asarray(Xt, dtype=np.float64)
        self.N, self.d = self.Xt.shape
        self.shape = (self.N, 2 * self.d + 2 * self.N)
        self.dtype = np.float64

    def _split(self, x):
        d, N = self.d, self.N
        return x[:d], x[d:2 * d], x[2 * d:2 * d + N], x[2 * d + N:]

    def __matmul__(self, x):
        """A x = Xt (w+ - w-) + xi - s   (x an n-vector or an n x k block)."""
        wp, wm, xi, s = self._split(x)
        return self.Xt @ (wp - wm) + xi - s

    def rmatmul(self, y):
        """A^T y = [Xt^T y; -Xt^T y; y; -y]."""
        g = self.Xt.T @ y
        return np.concatenate([g, -g, y, -y], axis=0)

    @property
    def T(self):
        return _Transposed(self)

    def normal_parts(self, dvec, delta):
        """(W, E) of N + delta I = Xt W Xt^T + diag(E)."""
        dwp, dwm, dxi, ds = self._split(dvec)
        return dwp + dwm, dxi + ds + delta

    def dense_normal_matrix(self, dvec, delta):
        """Materialised N + delta I (small instances only)."""
        W, E = self.normal_parts(dvec, delta)
        return (self.Xt * W[None, :]) @ self.Xt.T + np.diag(E)

    def direct_solver(self, dvec, delta):
        """Path D: exact solve with N + delta I through the Woodbury / capacitance identity."""
        W, E = self.normal_parts(dvec, delta)
        Einv = 1.0 / E
        XE = self.Xt * Einv[:, None]                          # E^{-1} Xt
        C = np.diag(1.0 / W) + self.Xt.T @ XE                 # W^{-1} + Xt^T E^{-1} Xt
        Cf = sla.cho_factor(C, lower=True)

        def solve(rhs, tol=None):
            u = Einv * rhs
            return u - XE @ sla.cho_solve(Cf, self.Xt.T @ u), {"iters": 0}
        return solve
