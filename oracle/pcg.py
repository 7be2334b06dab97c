"""Preconditioned conjugate gradient — ORACLE (test infrastructure only).

PAPER.md:220-235 (PCG on P^{-1/2}(N_k + delta_k I)P^{-1/2}); the Krylov.jl settings are not
given, so the loop below is the textbook PCG (Golub & Van Loan Alg. 11.5.1) with
  * zero initial guess unless x0 is given,
  * an ABSOLUTE stop on the recursively updated residual ||r||_2 <= tol_abs, checked before
    the first iteration and after every update, the true residual being
    recomputed once at exit and reported,
  * breakdown if p^T N p <= 0 or non-finite.
Iteration count = number of operator applications inside the loop.
"""
from __future__ import annotations

import numpy as np


class PCGBreakdown(RuntimeError):
    pass


def pcg(apply_op, rhs, apply_pinv=None, tol_abs=1e-10, max_iter=1000, x0=None, callback=None):
    rhs = np.asarray(rhs, dtype=np.float64)
    if apply_pinv is None:
        apply_pinv = lambda v: v  # noqa: E731  (P = I: plain CG)
    x = np.zeros_like(rhs) if x0 is None else np.array(x0, dtype=np.float64)
    r = rhs - apply_op(x) if x0 is not None else rhs.copy()
    it = 0
    rnorm = float(np.linalg.norm(r))
    converged = rnorm <= tol_abs
    if not converged:
        z = apply_pinv(r)
        p = z.copy()
        rz = float(r @ z)
        while it < max_iter:
            w = apply_op(p)
            pw = float(p @ w)
            if not np.isfinite(pw) or pw <= 0.0:
                raise PCGBreakdown(f"p^T N p = {pw} at iteration {it}")
            alpha = rz / pw
            x += alpha * p
            r -= alpha * w
            it += 1
            rnorm = float(np.linalg.norm(r))
            if callback is not None:
                callback(it, x, r)
            if rnorm <= tol_abs:
                converged = True
                break
            z = apply_pinv(r)
            rz_new = float(r @ z)
            beta = rz_new / rz
            p = z + beta * p
            rz = rz_new
    true_res = float(np.linalg.norm(rhs - apply_op(x)))
    return x, {"iters": it, "res": rnorm, "true_res": true_res, "converged": converged}
