"""Exact optimum of a separable QP with Q = diag(q) > 0 by dual semismooth Newton — ORACLE (test
infrastructure only).  An independent pin of f* for the IP-PMM oracle.

Problem (P)/(D) of PAPER.md:25-39 with Q = diag(q), every q_j > 0:
    min 1/2 x^T Q x + c^T x   s.t.  A x = b,  x >= 0.
Its Lagrangian dual is unconstrained (textbook: minimise the Lagrangian over x >= 0 coordinatewise):
    g(y) = b^T y + sum_j min_{x_j >= 0} (1/2 q_j x_j^2 + (c_j - a_j^T y) x_j)
         = b^T y - 1/2 sum_j max(0, a_j^T y - c_j)^2 / q_j,
concave and piecewise quadratic, with the primal point recovered in closed form
    x_j(y) = max(0, a_j^T y - c_j) / q_j,    grad g(y) = b - A x(y),
and a generalised Hessian  -A_S diag(1/q_S) A_S^T,  S = {j : a_j^T y > c_j}.  Strong duality holds
(Q > 0, feasible primal), so at the maximiser y*:  x(y*) is the unique primal optimum and
f* = 1/2 x*^T Q x* + c^T x* = g(y*).

Method: semismooth Newton on grad g = 0 with a Levenberg-Marquardt regulariser tau_k I,
tau_k = min(1e-4, ||grad g||) * (1 + max diag), so the system stays SPD when |S| < m, and an
Armijo backtracking line search on g (standard globalisation; e.g. Qi & Sun 1993 / Li, Sun & Toh
2018).  It shares nothing with IP-PMM: no barrier, no regularisation path, no Krylov solver.
Stops when ||b - A x(y)|| <= tol (1 + ||b||) and the Newton decrement is below rounding.

Exact KKT of the returned point (by construction of x(y)):
    x >= 0,  z = c + Q x - A^T y >= 0 with x_j z_j = 0 for every j (z_j = 0 where x_j > 0,
    z_j = c_j - a_j^T y >= 0 where x_j = 0);
only the primal residual b - A x is nonzero, reported as rel_p.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def dual_value(A, q, b, c, y):
    """g(y) = b^T y - 1/2 sum_j max(0, a_j^T y - c_j)^2 / q_j."""
    t = np.maximum(0.0, A.T @ y - c)
    return float(b @ y - 0.5 * np.sum(t * t / q))


def primal_of(A, q, c, y):
    """x_j(y) = max(0, a_j^T y - c_j) / q_j."""
    return np.maximum(0.0, A.T @ y - c) / q


def solve(A, q, b, c, tol=1e-14, max_iter=200, y0=None):
    A = np.asarray(A, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    if np.any(q <= 0):
        raise ValueError("semismooth Newton dual needs Q = diag(q) > 0")
    m, n = A.shape
    bnorm = float(np.linalg.norm(b))
    y = np.zeros(m) if y0 is None else np.array(y0, dtype=np.float64)
    g = dual_value(A, q, b, c, y)
    it = 0
    hist = []
    for it in range(max_iter):
        s = A.T @ y - c
        x = np.maximum(0.0, s) / q
        grad = b - A @ x
        gn = float(np.linalg.norm(grad))
        hist.append(gn)
        if gn <= tol * (1.0 + bnorm):
            break
        # rounding floor reached: the residual has not halved over the last 5 Newton steps
        if len(hist) > 6 and gn > 0.5 * min(hist[-6:-1]) and gn <= 1e-9 * (1.0 + bnorm):
            break
        S = s > 0
        AS = A[:, S]
        H = (AS / q[S][None, :]) @ AS.T                      # -(generalised Hessian)
        scale = 1.0 + float(np.max(np.diag(H))) if H.size else 1.0
        tau = min(1e-10 * scale, gn)
        H[np.diag_indices(m)] += tau
        dy = sla.cho_solve(sla.cho_factor(H, lower=True), grad)
        slope = float(grad @ dy)                              # > 0: ascent direction of g
        t = 1.0
        while True:
            yt = y + t * dy
            gt = dual_value(A, q, b, c, yt)
            if gt >= g + 1e-4 * t * slope or t < 1e-12:
                break
            t *= 0.5
        y, g = yt, gt
    x = primal_of(A, q, c, y)
    z = c + q * x - A.T @ y
    f = float(0.5 * x @ (q * x) + c @ x)
    rp = float(np.linalg.norm(b - A @ x)) / (1.0 + bnorm)
    return {"x": x, "y": y, "z": z, "obj": f, "dual_obj": dual_value(A, q, b, c, y), "rel_p": rp,
            "iters": it, "active": int(np.count_nonzero(x > 0))}
