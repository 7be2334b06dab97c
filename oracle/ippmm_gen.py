"""Nys-IP-PMM for QPs with FREE and BOX-CONSTRAINED variables, (P~)/(D~) — ORACLE (test infrastructure
only).  SURVEY §8(f) f1.

PAPER.md:771-846 (problem (P~)/(D~), Alg. 4 "Solve Newton system"), P:858-918 (Alg. 5 with w, s),
App. B.2 (initial point with u), App. B.3 (stepsizes with w, s).
Variable types: vtype[j] = 0 -> j in I (x_j >= 0), 1 -> F (free), 2 -> J (0 <= x_j <= u_j).
Vectors u, z, s, w have length n with u_IF = 0, z_F = 0, s_IF = 0, w_IF = 0.

  Theta^{-1}_j = z_j / x_j (j in IJ) + s_j / w_j (j in J), 0 on F   (from eq. P:1431 by elimination,
  reading G0: the paper's derivation gives -(Q + X^{-1}Z + W^{-1}S + rho I) dx + A^T dy = r_d + xi_au)
  xi_au (Alg. 4 line 1), xi = r_p + A D (r_d + xi_au), (N + delta I) dy = xi,
  dx = D (A^T dy - r_d - xi_au), dw_J = (r_u)_J - dx_J, dz_IJ = X^{-1} r_xz - Z dx (A15 reading:
  X^{-1}(r_xz - Z dx)), ds_J = W^{-1}(r_ws - S dw).

Readings where the paper is silent:
  G1 TC: rel_p = ||[b - A x; u_J - x_J - w_J]|| / (1 + ||[b; u_J]||), rel_d = ||c + Qx - A^T y - z + s|| /
     (1 + ||c||), mu (P:888 general) <= tol; the PEU "primal improved" test uses the same primal norm.
  G2 initial point: the delta~_d denominator read as sum(x~_IJ + delta_p) + sum(w~_J + delta_p) (A13).
  G3 the initial-point systems use (A A^T + 10 I) as in App. B.2; x~_F is not shifted.
  G5 with no inequality at all (every variable free) the duality measure and the corrector's target
     are 0 (the sums in P:882 / P:888 are empty): the iteration is the proximal method of multipliers
     on the equality-constrained QP.
"""
from __future__ import annotations

import numpy as np

from .ippmm import Options, Result, _krylov_solver, _direct_solver, _default_omega, build_preconditioner, \
    pcg_tolerance, peu_factor
from .linops import scaling_d  # noqa: F401  (documentation: the I-only special case)
from .rng import omega_stream


def masks(vtype):
    vt = np.asarray(vtype)
    I, F, J = vt == 0, vt == 1, vt == 2
    return I, F, J, I | J


def theta_inv(x, z, w, s, vtype):
    """Theta^{-1}: z/x on IJ, + s/w on J, 0 on F."""
    I, F, J, IJ = masks(vtype)
    t = np.zeros_like(x)
    t[IJ] = z[IJ] / x[IJ]
    t[J] += s[J] / w[J]
    return t


def mu_general(x, z, w, s, vtype):
    """mu = (x_IJ^T z_IJ + w_J^T s_J) / (|IJ| + |J|)   (P:888 / Alg. 5 line 4)."""
    I, F, J, IJ = masks(vtype)
    den = int(IJ.sum() + J.sum())
    return float(x[IJ] @ z[IJ] + w[J] @ s[J]) / den if den else 0.0


def stepsize_general(x, dx, w, dw, vtype):
    """alpha = 0.995 min{1, min_{I_x} -x/dx, min_{I_w} -w/dw}   (A16 for empty sets)."""
    I, F, J, IJ = masks(vtype)
    a = 1.0
    nx = IJ & (dx < 0)
    if nx.any():
        a = min(a, float(np.min(-x[nx] / dx[nx])))
    nw = J & (dw < 0)
    if nw.any():
        a = min(a, float(np.min(-w[nw] / dw[nw])))
    return 0.995 * a


def newton_direction_general(A, d, x, z, w, s, vtype, r_d, r_p, r_u, r_xz, r_ws, solve_normal):
    """Alg. 4."""
    I, F, J, IJ = masks(vtype)
    xi_au = np.zeros_like(x)
    xi_au[IJ] = -r_xz[IJ] / x[IJ]
    xi_au[J] += (r_ws[J] - s[J] * r_u[J]) / w[J]
    xi = r_p + A @ (d * (r_d + xi_au))
    dy, info = solve_normal(xi)
    dx = d * (A.T @ dy - r_d - xi_au)
    dw = np.zeros_like(x)
    dw[J] = r_u[J] - dx[J]
    dz = np.zeros_like(x)
    dz[IJ] = (r_xz[IJ] - z[IJ] * dx[IJ]) / x[IJ]
    ds = np.zeros_like(x)
    ds[J] = (r_ws[J] - s[J] * dw[J]) / w[J]
    info["xi_norm"] = float(np.linalg.norm(xi))
    return dx, dy, dz, dw, ds, info


def initial_point_general(A, q, b, c, vtype, u, solve_aat):
    """App. B.2."""
    I, F, J, IJ = masks(vtype)
    uu = np.where(J, u, 0.0)
    u1, _ = solve_aat(b - 0.5 * (A @ uu))
    xt = 0.5 * uu + A.T @ u1
    yt, _ = solve_aat(A @ (c + q * xt))
    g = c - A.T @ yt + q * xt
    zt = np.where(J, 0.5 * g, np.where(F, 0.0, g))             # z~_J = g_J / 2, z~_IF = g_IF (z_F := 0)
    st = np.where(J, -zt, 0.0)
    wt = np.where(J, uu - xt, 0.0)
    cand_p = [xt[IJ]] + ([wt[J]] if J.any() else [])
    cand_d = [zt[IJ]] + ([st[J]] if J.any() else [])
    dp = max([-1.5 * float(np.min(v)) for v in cand_p if v.size] + [0.0])      # P:1468 general (G5: none)
    dd = max([-1.5 * float(np.min(v)) for v in cand_d if v.size] + [0.0])
    gxz = float((xt[IJ] + dp) @ (zt[IJ] + dd))
    gws = float((wt[J] + dp) @ (st[J] + dd))
    den_p = float(np.sum(zt[IJ] + dd) + np.sum(st[J] + dd))
    den_d = float(np.sum(xt[IJ] + dp) + np.sum(wt[J] + dp))                  # G2
    dpt = dp + (0.5 * (gxz + gws) / den_p if den_p > 0 else 0.0)
    ddt = dd + (0.5 * (gxz + gws) / den_d if den_d > 0 else 0.0)
    x0 = np.where(IJ, xt + dpt, xt)
    w0 = np.where(J, wt + dpt, 0.0)
    z0 = np.where(IJ, zt + ddt, 0.0)
    s0 = np.where(J, st + ddt, 0.0)
    return x0, yt, z0, w0, s0


def solve_general(A, q, b, c, vtype, u, opts: Options = Options()) -> Result:
    """Alg. 3 / Alg. 5 for (P~)/(D~) with the Nystrom PCG path (opts.path = "krylov") or the dense
    direct path.  Returns Result with x, y, z (and w, s in log[-1]['w'], ['s'])."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    vtype = np.asarray(vtype, dtype=np.int64)
    I, F, J, IJ = masks(vtype)
    u = np.where(J, np.asarray(u, dtype=np.float64), 0.0)
    omega_fn = opts.omega_fn or _default_omega(opts.seed)
    max_iter = opts.pcg_max_iter
    bn = float(np.sqrt(b @ b + u[J] @ u[J]))
    cn = float(np.linalg.norm(c))

    ones = np.ones(n)
    if opts.path == "direct":
        sol0 = _direct_solver(A, ones, opts.init_delta)
        solve_aat = lambda r: sol0(r)  # noqa: E731
    else:
        U0 = lam0 = None
        if opts.ell > 0:
            U0, lam0, _ = build_preconditioner(A, ones, opts.ell, omega_fn(m, opts.ell, omega_stream(-1)))
        sol0 = _krylov_solver(A, ones, opts.init_delta, U0, lam0, max_iter)
        solve_aat = lambda r: sol0(r, opts.init_tol_rel * float(np.linalg.norm(r)))  # noqa: E731
    x, y, z, w, s = initial_point_general(A, q, b, c, vtype, u, solve_aat)

    lam_est, zeta = y.copy(), x.copy()
    rho, delta = opts.rho0, opts.delta0

    def residuals(x, y, z, w, s):
        rP = b - A @ x
        rU = np.where(J, u - x - w, 0.0)
        rD = c + q * x - A.T @ y - z + s
        return float(np.sqrt(rP @ rP + rU @ rU)), float(np.linalg.norm(rD))

    nrP, nrD = residuals(x, y, z, w, s)
    nrP_ref, nrD_ref = nrP, nrD
    mu = mu_general(x, z, w, s, vtype)
    log, status, inner_total, k = [], "max_outer", 0, 0
    for k in range(opts.max_outer + 1):
        rel_p, rel_d = nrP / (1.0 + bn), nrD / (1.0 + cn)
        if rel_p <= opts.tol and rel_d <= opts.tol and mu <= opts.tol:        # G1
            status = "optimal"
            break
        if k == opts.max_outer:
            break
        d = 1.0 / (q + theta_inv(x, z, w, s, vtype) + rho)
        if opts.path == "direct":
            sol = _direct_solver(A, d, delta)
        else:
            U = lamh = None
            if opts.ell > 0:
                U, lamh, _ = build_preconditioner(A, d, opts.ell, omega_fn(m, opts.ell, omega_stream(k)))
            sol = _krylov_solver(A, d, delta, U, lamh, max_iter)

        def solve_normal(xi, _sol=sol):
            return _sol(xi, pcg_tolerance(float(np.linalg.norm(xi)), mu, bn, opts.pcg_c, opts.pcg_floor))

        # predictor (eq. P:867-876)
        r_d = c + q * x - A.T @ y - z + s + rho * (x - zeta)
        r_p = b - A @ x - delta * (y - lam_est)
        r_u = np.where(J, u - x - w, 0.0)
        r_xz = np.where(IJ, -x * z, 0.0)
        r_ws = np.where(J, -w * s, 0.0)
        dxp, dyp, dzp, dwp, dsp, ip = newton_direction_general(A, d, x, z, w, s, vtype, r_d, r_p, r_u, r_xz, r_ws,
                                                              solve_normal)
        ap = stepsize_general(x, dxp, w, dwp, vtype)
        ad = stepsize_general(z, dzp, s, dsp, vtype)
        den = int(IJ.sum() + J.sum())
        if den == 0:             # G5: no inequality (all variables free): mu = mu_aff = mu~ = 0
            mu_aff = mu_t = 0.0
        else:
            mu_aff = float((x[IJ] + ap * dxp[IJ]) @ (z[IJ] + ad * dzp[IJ]) +
                           (w[J] + ap * dwp[J]) @ (s[J] + ad * dsp[J])) / den              # eq. P:882
            mu_t = mu_aff ** 3 / mu ** 2
        # corrector (eq. P:894-897)
        zn, zm = np.zeros(n), np.zeros(m)
        r_xz_c = np.where(IJ, mu_t - dxp * dzp, 0.0)
        r_ws_c = np.where(J, mu_t - dwp * dsp, 0.0)
        dxc, dyc, dzc, dwc, dsc, ic = newton_direction_general(A, d, x, z, w, s, vtype, zn, zm, zn, r_xz_c, r_ws_c,
                                                              solve_normal)
        dx, dy, dz, dw, ds = dxp + dxc, dyp + dyc, dzp + dzc, dwp + dwc, dsp + dsc
        ap = stepsize_general(x, dx, w, dw, vtype)
        ad = stepsize_general(z, dz, s, ds, vtype)
        x, w = x + ap * dx, w + ap * dw
        y, z, s = y + ad * dy, z + ad * dz, s + ad * ds
        mu_new = mu_general(x, z, w, s, vtype)
        nrP, nrD = residuals(x, y, z, w, s)
        # G5: mu = 0 (no inequality) -> the reduction is complete, r = 1
        r = min(max(1.0 - mu_new / mu, 0.0), 1.0) if mu > 0 else (1.0 if den == 0 else 0.0)
        p_imp, d_imp = nrP <= 0.95 * nrP_ref, nrD <= 0.95 * nrD_ref
        if p_imp:
            lam_est, nrP_ref = y.copy(), nrP
        if d_imp:
            zeta, nrD_ref = x.copy(), nrD
        delta = max(opts.reg_floor, peu_factor(p_imp, r) * delta)
        rho = max(opts.reg_floor, peu_factor(d_imp, r) * rho)
        it_p, it_c = ip.get("iters", 0), ic.get("iters", 0)
        inner_total += it_p + it_c
        log.append({"k": k, "mu": mu, "rel_p": rel_p, "rel_d": rel_d, "alpha_p": ap, "alpha_d": ad,
                    "pcg_pred": it_p, "pcg_corr": it_c, "w": w.copy(), "s": s.copy()})
        mu = mu_new
    obj = float(0.5 * x @ (q * x) + c @ x)
    dual_obj = float(b @ y - u[J] @ s[J] - 0.5 * x @ (q * x))
    res = Result(x, y, z, status, k, inner_total, obj, dual_obj, nrP / (1.0 + bn), nrD / (1.0 + cn), mu, log)
    res.w, res.s = w, s
    return res
