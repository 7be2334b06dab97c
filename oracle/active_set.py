"""Brute-force active-set enumeration for tiny separable QPs — ORACLE (test infrastructure only).

SPEC.md:535-543 ("enumerate_active_sets"): for every subset S of variables allowed to be
positive (the rest fixed at 0), solve the equality-constrained KKT system densely,
    [Q_S  -A_S^T] [x_S]   [-c_S]
    [A_S    0   ] [ y ] = [  b ]
and keep candidates satisfying the KKT conditions of (P)/(D):
    A x = b, x >= 0, z = c + Q x - A^T y >= 0, z_S = 0.
For a convex QP any KKT point is optimal; the minimum-objective candidate is returned.
Independent of the IP-PMM oracle (no interior-point arithmetic at all).
"""
from __future__ import annotations

import itertools

import numpy as np


def enumerate_active_sets(A, q, b, c, tol=1e-9):
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    best = None
    for k in range(0, n + 1):
        for S in itertools.combinations(range(n), k):
            S = list(S)
            nS = len(S)
            K = np.zeros((nS + m, nS + m))
            rhs = np.zeros(nS + m)
            if nS:
                K[:nS, :nS] = np.diag(q[S])
                K[:nS, nS:] = -A[:, S].T
                K[nS:, :nS] = A[:, S]
                rhs[:nS] = -c[S]
            rhs[nS:] = b
            sol, *_ = np.linalg.lstsq(K, rhs, rcond=None)
            if np.linalg.norm(K @ sol - rhs) > tol * (1.0 + np.linalg.norm(rhs)):
                continue
            x = np.zeros(n)
            x[S] = sol[:nS]
            y = sol[nS:]
            if np.min(x, initial=0.0) < -tol:
                continue
            z = c + q * x - A.T @ y
            if np.min(z, initial=0.0) < -tol * (1.0 + np.abs(c).max()):
                continue
            if np.linalg.norm(A @ x - b) > 1e-8 * (1.0 + np.linalg.norm(b)):
                continue
            f = 0.5 * x @ (q * x) + c @ x
            if best is None or f < best[0] - 1e-12:
                best = (f, x, y, np.maximum(z, 0.0))
    if best is None:
        raise RuntimeError("no KKT point found (infeasible or unbounded)")
    f, x, y, z = best
    return {"obj": float(f), "x": x, "y": y, "z": z}


def enumerate_active_sets_general(A, q, b, c, vtype, u, tol=1e-9):
    """Brute force for tiny (P~): every variable of I is at 0 or free (> 0), every variable
    of J at 0, at u_j or strictly between, every variable of F free; solve the KKT system of the
    resulting equality-constrained QP and keep the best point that is primal and dual feasible
    (z = c + Qx - A^T y >= 0 at lower bounds, <= 0 at upper bounds, = 0 in between)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    vtype = np.asarray(vtype)
    choices = [((0, "free") if t == 0 else (("free",) if t == 1 else (0, "ub", "free"))) for t in vtype]
    best = None
    for combo in itertools.product(*choices):
        fixed = {j: (0.0 if s == 0 else u[j]) for j, s in enumerate(combo) if s != "free"}
        S = [j for j in range(n) if j not in fixed]
        nS = len(S)
        xf = np.zeros(n)
        for j, v in fixed.items():
            xf[j] = v
        K = np.zeros((nS + m, nS + m))
        rhs = np.zeros(nS + m)
        if nS:
            K[:nS, :nS] = np.diag(q[S])
            K[:nS, nS:] = -A[:, S].T
            K[nS:, :nS] = A[:, S]
            rhs[:nS] = -c[S]
        rhs[nS:] = b - A @ xf
        sol, *_ = np.linalg.lstsq(K, rhs, rcond=None)
        if np.linalg.norm(K @ sol - rhs) > tol * (1.0 + np.linalg.norm(rhs)):
            continue
        x = xf.copy()
        x[S] = sol[:nS]
        y = sol[nS:]
        ok = True
        g = c + q * x - A.T @ y
        sc = tol * (1.0 + np.abs(c).max())
        for j in range(n):
            st = combo[j]
            if vtype[j] != 1 and x[j] < -tol:
                ok = False
            if vtype[j] == 2 and x[j] > u[j] + tol:
                ok = False
            if st == 0 and g[j] < -sc:
                ok = False
            if st == "ub" and g[j] > sc:
                ok = False
        if not ok or np.linalg.norm(A @ x - b) > 1e-8 * (1.0 + np.linalg.norm(b)):
            continue
        f = 0.5 * x @ (q * x) + c @ x
        if best is None or f < best[0] - 1e-12:
            best = (f, x, y)
    if best is None:
        raise RuntimeError("no KKT point found")
    return {"obj": float(best[0]), "x": best[1], "y": best[2]}
