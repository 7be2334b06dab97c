"""Nys-IP-PMM for the separable QP pair (P)/(D) with x >= 0 — ORACLE (test infrastructure only).

Specialisation of Alg. 3, Alg. 4 and Alg. 5 to
F = J = {} (every BASELINE config is x >= 0 only), with the initial point of App. B.2
(u = 0) and the stepsizes of App. B.3.

Two solve paths for the normal equations (N_k + delta_k I) dy = xi:
  path "direct": dense Cholesky of A D A^T + delta I (reused by predictor and corrector)
  path "krylov": PCG (oracle.pcg) with P = I (ell = 0) or the Nystrom P^{-1} of Alg. 2.

Readings where the paper defers to external algorithms or is silent:
  A8'  PCG tolerance tau_k = max(1e-10 (1+||b||), min(0.1 ||xi||, 1e-3 mu_k (1+||b||)))
       (absolute, on the recursive residual; tracks ||theta|| <= C mu_k of Prop. 3.1, P:685-693;
       the constants are unpinned, chosen in DESIGN.md from a sweep on configs 0/1/3)
  A10' PCG max_iter = 20000; on exhaustion the direction is accepted (inexact IP-PMM)
  A11  TC: ||b-Ax||/(1+||b||) <= tol, ||c+Qx-A^T y-z||/(1+||c||) <= tol, mu <= tol
  A12  PEU: r = clip(1 - mu+/mu, 0, 1); primal "improved" iff ||r_P+|| <= 0.95 ||r_P at last
       lambda update||, then lambda <- y+, delta <- max(5e-10, (1-r) delta), else
       delta <- max(5e-10, (1 - 2/3 r) delta); dual likewise with zeta <- x+, rho.
       (form pinned by Tables 5-6; the 0.95 test itself is unpinned)
  A13  initial point: delta~_d denominator read as sum(x~ + delta_p)
  A14'' initial-point PCG tolerance 1e-12 ||rhs|| (tighter than SURVEY A14; at 1e-8 the
       initial point depended on Omega at ~1e-6 on the config-1 recipe, at 1e-12 at ~1e-10: the
       initial point is then a property of the problem, not of the Krylov rounding)
  A15  dz = X^{-1}(r_xz - Z dx)
  A16  empty ratio-test set -> alpha = 0.995
  IPg  initial-point guard: if a shifted x0 (z0) still has a non-positive entry (only when
       gamma = 0), add 1 to delta~_p (delta~_d).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import scipy.linalg as sla

from .linops import normal_matvec, scaling_d, sketch, dense_normal_matrix
from .nystrom import nystrom_from_sketch, precond_inv_apply
from .partial_chol import partial_cholesky, chol_precond_inv_apply
from .pcg import pcg
from .rng import gaussian_omega, omega_stream


@dataclass
class Options:
    tol: float = 1e-8
    ell: int = 0                       # fixed sketch size; 0 = CG-IP-PMM
    path: str = "krylov"               # "krylov" | "direct"
    seed: int = 0
    max_outer: int = 100
    rho0: float = 8.0
    delta0: float = 8.0
    reg_floor: float = 5e-10           # Tables 5-6 floor
    pcg_c: float = 1e-3                # A8'
    pcg_floor: float = 1e-10           # A8'
    pcg_max_iter: int = 20000          # A10'
    init_delta: float = 10.0
    init_tol_rel: float = 1e-12        # A14''
    omega_fn: Optional[Callable[[int, int, int], np.ndarray]] = None  # (m, ell, stream) -> Omega
    # preconditioner reuse ("reusing the preconditioner between iterations"):
    # rebuild when k - k_last >= prec_refresh, or when the previous iteration's PCG count exceeded
    # prec_growth x the count right after the last rebuild; (1, 0.0) = Alg. 3 as written
    prec_refresh: int = 1
    prec_growth: float = 0.0
    # "nystrom" (Nys-IP-PMM) or "chol": the partial Cholesky preconditioner of rank ell (Chol-IP-PMM,
    # the paper's comparison arm), rebuilt every outer iteration
    precond: str = "nystrom"
    # adaptive rank (the paper's future work "tuning the rank"; reading F1 in
    # DESIGN.md): when ell_max > ell, after a Nystrom build with rank ell_k whose estimate
    # lam_hat_ell exceeds ell_tau * mu_prec (mu_prec = delta_k, A7), the next build uses
    # min(2 ell_k, ell_max) (a rebuild is forced at the next iteration); the rank never shrinks
    ell_max: int = 0
    ell_tau: float = 10.0


@dataclass
class Result:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    status: str
    outer: int
    inner_total: int
    obj: float
    dual_obj: float
    rel_p: float
    rel_d: float
    mu: float
    log: list = field(default_factory=list)


# ----------------------------------------------------------------------------------------
# building blocks
# ----------------------------------------------------------------------------------------

def stepsize(v, dv):
    """alpha = 0.995 min{1, min_{dv_i < 0} -v_i/dv_i}   (A16)."""
    neg = dv < 0
    if not np.any(neg):
        return 0.995
    return 0.995 * min(1.0, float(np.min(-v[neg] / dv[neg])))


def duality_measure(x, z):
    """mu = x^T z / n   (P:888 with J = {})."""
    return float(x @ z) / x.shape[0]


def peu_factor(improved: bool, r: float) -> float:
    """A12: multiplicative update of delta (primal) / rho (dual)."""
    return (1.0 - r) if improved else (1.0 - (2.0 / 3.0) * r)


def pcg_tolerance(xi_norm, mu, b_norm, c=1e-3, floor=1e-10):
    """A8': tau_k = max(floor (1+||b||), min(0.1 ||xi||, c mu_k (1+||b||)))."""
    return max(floor * (1.0 + b_norm), min(0.1 * xi_norm, c * mu * (1.0 + b_norm)))


def newton_direction(A, d, x, z, r_d, r_p, r_xz, solve_normal):
    """Alg. 4 for I-only variables.

    xi_au = -X^{-1} r_xz ; xi = r_p + A D (r_d + xi_au) ; (N + delta I) dy = xi ;
    dx = D (A^T dy - r_d - xi_au) ; dz = X^{-1}(r_xz - Z dx)   (A15)
    """
    xi_au = -r_xz / x
    xi = r_p + A @ (d * (r_d + xi_au))
    dy, info = solve_normal(xi)
    dx = d * (A.T @ dy - r_d - xi_au)
    dz = (r_xz - z * dx) / x
    info["xi_norm"] = float(np.linalg.norm(xi))
    return dx, dy, dz, xi, info


def newton_block_residuals(A, q, rho, delta, x, z, dx, dy, dz, r_d, r_p, r_xz):
    """Residuals of the 3-block Newton system for a direction (Prop. 3.1 test)."""
    b1 = -(q + rho) * dx + A.T @ dy + dz - r_d
    b2 = A @ dx + delta * dy - r_p
    b3 = z * dx + x * dz - r_xz
    return b1, b2, b3


def initial_point(A, q, b, c, solve_aat):
    """App. B.2 with u = 0, F = J = {}.

    solve_aat(rhs) solves (A A^T + 10 I) u = rhs (P:1464 regularisation delta = 10).
    """
    u1, i1 = solve_aat(b)
    xt = A.T @ u1                                           # x~ = A^T (AA^T)^{-1} b
    yt, i2 = solve_aat(A @ (c + q * xt))                    # y~ = (AA^T)^{-1} A (c + Q x~)
    zt = c - A.T @ yt + q * xt                              # z~
    dp = max(-1.5 * float(np.min(xt)), 0.0)
    dd = max(-1.5 * float(np.min(zt)), 0.0)
    gamma = float((xt + dp) @ (zt + dd))
    sz = float(np.sum(zt + dd))
    sx = float(np.sum(xt + dp))                             # A13
    dpt = dp + (0.5 * gamma / sz if sz > 0 else 0.0)
    ddt = dd + (0.5 * gamma / sx if sx > 0 else 0.0)
    x0 = xt + dpt
    z0 = zt + ddt
    if np.min(x0) <= 0.0:                                   # IPg
        x0 = xt + (dpt + 1.0)
    if np.min(z0) <= 0.0:
        z0 = zt + (ddt + 1.0)
    return x0, yt.copy(), z0, {"pcg_iters": i1.get("iters", 0) + i2.get("iters", 0)}


# ----------------------------------------------------------------------------------------
# normal-equation solvers (path D / path K)
# ----------------------------------------------------------------------------------------

def _direct_solver(A, d, delta):
    if hasattr(A, "direct_solver"):            # structured operator (oracle.svm): Woodbury path D
        return A.direct_solver(d, delta)
    L = sla.cho_factor(dense_normal_matrix(A, d, delta), lower=True)

    def solve(rhs, tol=None):
        return sla.cho_solve(L, rhs), {"iters": 0}
    return solve


def _krylov_solver(A, d, delta, U, lam, max_iter, chol=None):
    apply_op = lambda v: normal_matvec(A, d, v, delta)  # noqa: E731
    if chol is not None:
        pinv = lambda v: chol_precond_inv_apply(chol, v)  # noqa: E731
    elif U is None:
        pinv = None
    else:
        pinv = lambda v: precond_inv_apply(U, lam, delta, v)  # noqa: E731 (mu_prec = delta, A7)

    def solve(rhs, tol):
        x, info = pcg(apply_op, rhs, pinv, tol_abs=tol, max_iter=max_iter)
        return x, info
    return solve


def _default_omega(seed):
    def fn(m, ell, stream):
        return gaussian_omega(m, ell, seed, stream)
    return fn


def build_preconditioner(A, d, ell, Omega):
    """Alg. 2: Nystrom factors of N_k = A D A^T from the sketch Y = N_k Omega."""
    Y = sketch(A, d, Omega)
    U, lam, info = nystrom_from_sketch(Y, Omega)
    return U, lam, info


# ----------------------------------------------------------------------------------------
# Alg. 3 outer loop
# ----------------------------------------------------------------------------------------

def solve(A, q, b, c, opts: Options = Options()) -> Result:
    """A: dense m x n array, or a structured operator with @, .T @, .shape and direct_solver
    (oracle.svm.SvmOperator: config 2 without materialising its 40.8 GB A)."""
    if not hasattr(A, "direct_solver"):
        A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    omega_fn = opts.omega_fn or _default_omega(opts.seed)
    max_iter = opts.pcg_max_iter
    bnorm = float(np.linalg.norm(b))
    cnorm = float(np.linalg.norm(c))

    # ---- initial point (App. B.2) ------------------------------------------------
    ones = np.ones(n)
    if opts.path == "direct":
        sol0 = _direct_solver(A, ones, opts.init_delta)
        solve_aat = lambda r: sol0(r)  # noqa: E731
    else:
        U0 = lam0 = F0 = None
        if opts.ell > 0 and opts.precond == "chol":
            F0 = partial_cholesky(A, ones, opts.init_delta, opts.ell)
        elif opts.ell > 0:
            U0, lam0, _ = build_preconditioner(A, ones, opts.ell, omega_fn(m, opts.ell, omega_stream(-1)))
        sol0 = _krylov_solver(A, ones, opts.init_delta, U0, lam0, max_iter, F0)
        solve_aat = lambda r: sol0(r, opts.init_tol_rel * float(np.linalg.norm(r)))  # noqa: E731
    x, y, z, info0 = initial_point(A, q, b, c, solve_aat)
    inner_total = info0["pcg_iters"]

    # ---- PMM parameters ----------------------------------------------------------
    lam_est, zeta = y.copy(), x.copy()
    rho, delta = opts.rho0, opts.delta0
    rP = b - A @ x
    rD = c + q * x - A.T @ y - z
    nrP, nrD = float(np.linalg.norm(rP)), float(np.linalg.norm(rD))
    nrP_ref, nrD_ref = nrP, nrD
    mu = duality_measure(x, z)
    log = []
    status = "max_outer"
    k = 0
    U = lamh = None
    last_build, base_its, last_its = -1, None, 0
    ell_k = opts.ell                       # rank of the next Nystrom build (F1)
    ell_built = opts.ell                   # rank of the factors in use
    for k in range(opts.max_outer + 1):
        rel_p, rel_d = nrP / (1.0 + bnorm), nrD / (1.0 + cnorm)
        # ---- TC (A11) ----
        if rel_p <= opts.tol and rel_d <= opts.tol and mu <= opts.tol:
            status = "optimal"
            break
        if k == opts.max_outer:
            break
        # ---- N_k as an operator ----
        d = scaling_d(q, x, z, rho)
        delta_used = delta
        # ---- P_k^{-1} ----
        if opts.path == "direct":
            sol = _direct_solver(A, d, delta)
        else:
            built = False
            F = None
            if opts.ell > 0 and opts.precond == "chol":
                F = partial_cholesky(A, d, delta, opts.ell)               # P:250-349, every iteration
                built = True
            elif opts.ell > 0:
                rebuild = (last_build < 0 or k - last_build >= max(1, opts.prec_refresh) or
                           (opts.prec_growth > 0 and base_its and last_its > opts.prec_growth * base_its) or
                           ell_k != ell_built)
                if rebuild:
                    U, lamh, _ = build_preconditioner(A, d, ell_k, omega_fn(m, ell_k, omega_stream(k)))
                    last_build, base_its, built, ell_built = k, None, True, ell_k
                    cap = min(opts.ell_max, m, 1024)
                    if cap > ell_k and lamh[ell_k - 1] > opts.ell_tau * delta:      # F1
                        ell_k = min(2 * ell_k, cap)
            sol = _krylov_solver(A, d, delta, U, lamh, max_iter, F)   # Nystrom: mu_prec = delta_k (A7)

        # ---- Alg. 5 predictor ----
        r_d = c + q * x - A.T @ y - z + rho * (x - zeta)
        r_p = b - A @ x - delta * (y - lam_est)
        r_xz = -x * z

        def solve_normal(xi, _sol=sol):
            tol = pcg_tolerance(float(np.linalg.norm(xi)), mu, bnorm, opts.pcg_c, opts.pcg_floor)
            return _sol(xi, tol)

        dxp, dyp, dzp, _, ip = newton_direction(A, d, x, z, r_d, r_p, r_xz, solve_normal)
        ap, ad = stepsize(x, dxp), stepsize(z, dzp)
        mu_aff = float((x + ap * dxp) @ (z + ad * dzp)) / n
        mu_t = mu_aff ** 3 / mu ** 2
        # ---- corrector ----
        zero_n, zero_m = np.zeros(n), np.zeros(m)
        r_xz_c = mu_t - dxp * dzp
        dxc, dyc, dzc, _, ic = newton_direction(A, d, x, z, zero_n, zero_m, r_xz_c, solve_normal)
        dx, dy, dz = dxp + dxc, dyp + dyc, dzp + dzc
        ap, ad = stepsize(x, dx), stepsize(z, dz)
        x = x + ap * dx
        y = y + ad * dy
        z = z + ad * dz
        mu_new = duality_measure(x, z)
        # ---- residuals at the new iterate (reused by TC next iteration) ----
        rP = b - A @ x
        rD = c + q * x - A.T @ y - z
        nrP, nrD = float(np.linalg.norm(rP)), float(np.linalg.norm(rD))
        # ---- PEU (A12) ----
        r = min(max(1.0 - mu_new / mu, 0.0), 1.0) if mu > 0 else 0.0
        p_imp = nrP <= 0.95 * nrP_ref
        d_imp = nrD <= 0.95 * nrD_ref
        if p_imp:
            lam_est = y.copy()
            nrP_ref = nrP
        if d_imp:
            zeta = x.copy()
            nrD_ref = nrD
        delta = max(opts.reg_floor, peu_factor(p_imp, r) * delta)
        rho = max(opts.reg_floor, peu_factor(d_imp, r) * rho)
        it_p, it_c = ip.get("iters", 0), ic.get("iters", 0)
        inner_total += it_p + it_c
        last_its = it_p + it_c
        if base_its is None:
            base_its = last_its
        log.append({"k": k, "mu": mu, "rel_p": rel_p, "rel_d": rel_d, "alpha_p": ap, "alpha_d": ad,
                    "pcg_pred": it_p, "pcg_corr": it_c, "rho_next": rho, "delta_next": delta,
                    "prec_built": bool(opts.path != "direct" and opts.ell > 0 and built),
                    "ell": ell_built if (opts.path != "direct" and opts.ell > 0 and opts.precond != "chol") else opts.ell,
                    "lam_ell": float(lamh[-1]) if lamh is not None else 0.0, "delta": delta_used,
                    "mu_next": mu_new})
        mu = mu_new

    obj = float(0.5 * x @ (q * x) + c @ x)
    dual_obj = float(b @ y - 0.5 * x @ (q * x))
    return Result(x, y, z, status, k, inner_total, obj, dual_obj,
                  nrP / (1.0 + bnorm), nrD / (1.0 + cnorm), mu, log)
