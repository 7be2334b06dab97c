"""Pins of the CPU oracle against what the paper and mathematics fix (runs without a GPU).

Each test names the passage it pins (P:n = PAPER.md line n, S:n = SPEC.md line n).
None of these re-types the oracle's own formula: they use closed forms, exact rational
arithmetic, brute force, textbook invariants or printed paper values.
"""
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import ippmm, linops, nystrom, pcg as pcgmod, rng
from oracle.active_set import enumerate_active_sets
from synth import make_config

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_psd_lowrank(rs, m, r, spread=1.0):
    Q, _ = np.linalg.qr(rs.standard_normal((m, r)))
    ev = np.logspace(0, -spread, r) * 3.0
    return (Q * ev) @ Q.T, Q, ev


# ------------------------------------------------------------------ normal operator
def test_normal_matvec_spec_example_s57():
    # A=[[1,1]], q=0, theta^{-1}=1, rho=0, delta=0.5, v=(1) -> 2.5 (hand arithmetic: 1+1+0.5)
    A = np.array([[1.0, 1.0]])
    d = linops.scaling_d(np.zeros(2), np.ones(2), np.ones(2), 0.0)  # z/x = theta^{-1} = 1
    w = linops.normal_matvec(A, d, np.array([1.0]), 0.5)
    assert w[0] == 2.5


def test_normal_matvec_spec_example_s56_corrected():
    # S:56 with A=I2, q=(1,1), theta^{-1}=(1,1), rho=0, delta=1, v=(2,2):
    # d = 1/(1+1) = 1/2, so w = 1/2*2 + 1*2 = 3 (SPEC's printed (2,2) is wrong).
    d = linops.scaling_d(np.ones(2), np.ones(2), np.ones(2), 0.0)
    w = linops.normal_matvec(np.eye(2), d, np.array([2.0, 2.0]), 1.0)
    np.testing.assert_array_equal(w, [3.0, 3.0])


def test_normal_matvec_exact_rational():
    # brute force in exact rational arithmetic on a tiny instance (different arithmetic path)
    rs = np.random.default_rng(11)
    m, n = 5, 7
    A = rs.standard_normal((m, n))
    d = rs.uniform(0.1, 3.0, n)
    e = rs.uniform(0.0, 1.0, m)
    v = rs.standard_normal(m)
    delta = 0.37
    F = Fraction
    exact = []
    for i in range(m):
        s = F(0)
        for j in range(n):
            t = sum(F(A[k, j]) * F(v[k]) for k in range(m)) * F(d[j])
            s += F(A[i, j]) * t
        s += F(e[i]) * F(v[i]) + F(delta) * F(v[i])
        exact.append(float(s))
    exact = np.array(exact)
    w = linops.normal_matvec(A, d, v, delta, e)
    assert np.linalg.norm(w - exact) <= 1e-15 * np.linalg.norm(exact)


def test_sketch_columns_are_matvecs_without_delta():
    # Alg. 1 line 2 with SURVEY A1: Y = N_k Omega, N_k excludes delta
    inst = make_config(0)
    rs = np.random.default_rng(1)
    d = rs.uniform(0.1, 2.0, inst.n)
    Om = rs.standard_normal((inst.m, 5))
    Y = linops.sketch(inst.A, d, Om)
    for j in range(5):
        col = linops.normal_matvec(inst.A, d, Om[:, j], 1.0) - Om[:, j]
        assert np.linalg.norm(Y[:, j] - col) <= 1e-13 * np.linalg.norm(col)


def test_operator_is_spd_with_delta_floor():
    # <v, (N + delta I) v> >= delta ||v||^2
    inst = make_config(0)
    rs = np.random.default_rng(2)
    d = rs.uniform(0.0, 2.0, inst.n)
    for _ in range(50):
        v = rs.standard_normal(inst.m)
        assert v @ linops.normal_matvec(inst.A, d, v, 0.3) >= 0.3 * (v @ v) * (1 - 1e-14)


# ------------------------------------------------------------------ Nystrom (Alg. 1)
def test_nu_is_julia_eps_of_frobenius_norm():
    # P:376 nu = eps(norm(Y,'fro')) -- Julia eps(x) is the ulp spacing: 2^(floor(log2 x) - 52)
    Y = np.full((4, 2), 3.0)  # ||Y||_F = 6*sqrt(2) = 8.485..., floor(log2) = 3
    Om = np.eye(4)[:, :2]
    _, _, info = nystrom.nystrom_from_sketch(Y + 10 * np.eye(4)[:, :2], Om)
    Yf = np.linalg.norm(Y + 10 * np.eye(4)[:, :2], "fro")
    assert info["nu"] == 2.0 ** (np.floor(np.log2(Yf)) - 52)


def test_nystrom_identity_gives_unit_eigenvalues():
    # N = I5, l = 3 -> lambda_hat = (1,1,1)
    rs = np.random.default_rng(3)
    Om = rs.standard_normal((5, 3))
    U, lam, _ = nystrom.nystrom_from_sketch(Om.copy(), Om)
    np.testing.assert_allclose(lam, 1.0, atol=1e-12)
    np.testing.assert_allclose(U.T @ U, np.eye(3), atol=1e-13)


def test_nystrom_rank2_example_s167():
    # N = U diag(3,2,0,0) U^T, l = 2 -> lambda_hat = (3,2), N_hat = N
    rs = np.random.default_rng(4)
    Q, _ = np.linalg.qr(rs.standard_normal((4, 4)))
    N = (Q[:, :2] * [3.0, 2.0]) @ Q[:, :2].T
    Om = rs.standard_normal((4, 2))
    U, lam, _ = nystrom.nystrom_from_sketch(N @ Om, Om)
    np.testing.assert_allclose(lam, [3.0, 2.0], rtol=1e-12)
    np.testing.assert_allclose((U * lam) @ U.T, N, atol=1e-12)


@pytest.mark.parametrize("extra", [2, 10])
def test_nystrom_exact_recovery_above_rank(extra):
    # Nystrom approximation is exact when l > rank(N) (range(Y) = range(N))
    rs = np.random.default_rng(5)
    m, r = 60, 8
    N, _, _ = _rand_psd_lowrank(rs, m, r, spread=3)
    Om = rs.standard_normal((m, r + extra))
    U, lam, _ = nystrom.nystrom_from_sketch(N @ Om, Om)
    err = np.linalg.norm(N - (U * lam) @ U.T) / np.linalg.norm(N)
    assert err <= 1e-11
    np.testing.assert_allclose(U.T @ U, np.eye(r + extra), atol=1e-12)


def test_nystrom_is_below_N_in_loewner_order():
    # N_hat = Y (Omega^T Y)^+ Y^T is a projection of N: 0 <= N_hat <= N (Loewner)
    rs = np.random.default_rng(6)
    m = 40
    B = rs.standard_normal((m, m))
    N = B @ np.diag(np.logspace(0, -6, m)) @ B.T
    for ell in (3, 10, 25):
        Om = rs.standard_normal((m, ell))
        U, lam, _ = nystrom.nystrom_from_sketch(N @ Om, Om)
        assert np.all(lam >= 0) and np.all(np.diff(lam) <= 0)
        ev = np.linalg.eigvalsh(N - (U * lam) @ U.T)
        assert ev.min() >= -1e-12 * np.linalg.norm(N, 2)


def test_nystrom_matches_pseudoinverse_formula_on_wellconditioned_case():
    # eq.: N_hat = Y (Omega^T Y)^+ Y^T (the unstable textbook formula is fine when
    # Omega^T Y is well conditioned)
    rs = np.random.default_rng(7)
    m, ell = 30, 6
    B = rs.standard_normal((m, m))
    N = B @ B.T / m + np.eye(m)
    Om = rs.standard_normal((m, ell))
    Y = N @ Om
    ref = Y @ np.linalg.pinv(Om.T @ Y) @ Y.T
    U, lam, info = nystrom.nystrom_from_sketch(Y, Om)
    # lambda_hat subtracts nu: compare with the nu-shifted reference within nu-scale
    assert np.linalg.norm((U * lam) @ U.T - ref) <= 1e-10 * np.linalg.norm(ref)


# ------------------------------------------------------------------ preconditioner
def _factors(seed=8, m=50, ell=7):
    rs = np.random.default_rng(seed)
    B = rs.standard_normal((m, m))
    N = B @ np.diag(np.logspace(2, -3, m)) @ B.T
    Om = rs.standard_normal((m, ell))
    U, lam, _ = nystrom.nystrom_from_sketch(N @ Om, Om)
    return N, U, lam, rs


def test_precond_inverse_times_precond_is_identity():
    N, U, lam, rs = _factors()
    mu = 0.05
    for _ in range(5):
        v = rs.standard_normal(N.shape[0])
        w = nystrom.precond_inv_apply(U, lam, mu, nystrom.precond_apply(U, lam, mu, v))
        assert np.linalg.norm(w - v) <= 1e-12 * np.linalg.norm(v)


def test_precond_inverse_fixed_directions():
    # P^{-1} u_l = u_l; v orthogonal to range(U) -> P^{-1} v = v
    N, U, lam, rs = _factors()
    mu = 0.2
    ul = U[:, -1]
    np.testing.assert_allclose(nystrom.precond_inv_apply(U, lam, mu, ul), ul, atol=1e-13)
    v = rs.standard_normal(N.shape[0])
    v -= U @ (U.T @ v)
    np.testing.assert_allclose(nystrom.precond_inv_apply(U, lam, mu, v), v, atol=1e-13)


def test_precond_inverse_spectrum_range():
    # eig(P^{-1}) in [(lam_l+mu)/(lam_1+mu), 1]
    N, U, lam, _ = _factors()
    mu = 0.01
    ev = np.linalg.eigvalsh(nystrom.precond_inv_dense(U, lam, mu))
    lo = (lam[-1] + mu) / (lam[0] + mu)
    assert ev.min() >= lo * (1 - 1e-10) and ev.max() <= 1 + 1e-10


def test_preconditioned_condition_number_bound():
    # kappa(P^{-1/2} N_delta P^{-1/2}) <= (lam_l + delta + ||N - N_hat||_2)/delta
    N, U, lam, _ = _factors(m=60, ell=10)
    delta = 1e-2
    Nd = N + delta * np.eye(N.shape[0])
    Pi = nystrom.precond_inv_dense(U, lam, delta)
    w, V = np.linalg.eigh(Pi)
    S = (V * np.sqrt(w)) @ V.T
    ev = np.linalg.eigvalsh(S @ Nd @ S)
    kappa = ev.max() / ev.min()
    bound = (lam[-1] + delta + np.linalg.norm(N - (U * lam) @ U.T, 2)) / delta
    assert kappa <= bound * (1 + 1e-8)


def test_pcg_one_iteration_when_sketch_exceeds_rank():
    # l > rank(N): P^{-1}(N + delta I) = (lam_l+delta) I  -> PCG converges in one step
    rs = np.random.default_rng(9)
    m, r = 40, 5
    N, _, _ = _rand_psd_lowrank(rs, m, r, spread=4)
    Om = rs.standard_normal((m, r + 3))
    U, lam, _ = nystrom.nystrom_from_sketch(N @ Om, Om)
    delta = 1e-3
    b = rs.standard_normal(m)
    x, info = pcgmod.pcg(lambda v: N @ v + delta * v, b,
                         lambda v: nystrom.precond_inv_apply(U, lam, delta, v),
                         tol_abs=1e-10 * np.linalg.norm(b), max_iter=50)
    assert info["iters"] <= 2  # 1 in exact arithmetic; lam_hat carries nu-level noise
    assert np.linalg.norm(N @ x + delta * x - b) <= 1e-9 * np.linalg.norm(b)


def test_table2_matvec_cost():
    # Table 2: Nystrom P^{-1} matvec costs 2 l m + m + 5 l flops
    assert nystrom.precond_apply_flops(2000, 50) == 2 * 50 * 2000 + 2000 + 5 * 50


# ------------------------------------------------------------------ PCG
def test_pcg_identity_one_iteration():
    b = np.array([1.0, -2.0, 3.0])
    x, info = pcgmod.pcg(lambda v: v, b, tol_abs=1e-14)
    assert info["iters"] == 1
    np.testing.assert_allclose(x, b)


def test_pcg_three_distinct_eigenvalues():
    # diag(1,2,3) converges in <= 3 iterations (CG finite termination)
    Dg = np.array([1.0, 2.0, 3.0])
    b = np.random.default_rng(10).standard_normal(3)
    x, info = pcgmod.pcg(lambda v: Dg * v, b, tol_abs=1e-12)
    assert info["iters"] <= 3
    np.testing.assert_allclose(x, b / Dg, rtol=1e-12)


def test_pcg_perfect_preconditioner():
    rs = np.random.default_rng(11)
    B = rs.standard_normal((20, 20))
    M = B @ B.T + np.diag(np.logspace(0, 4, 20))
    Mi = np.linalg.inv(M)
    b = rs.standard_normal(20)
    x, info = pcgmod.pcg(lambda v: M @ v, b, lambda v: Mi @ v, tol_abs=1e-9 * np.linalg.norm(b))
    assert info["iters"] == 1


def test_pcg_energy_error_monotone_and_solution():
    # the energy-norm error is nonincreasing; result matches a dense solve
    rs = np.random.default_rng(12)
    B = rs.standard_normal((25, 25))
    M = B @ B.T + 0.1 * np.eye(25)
    b = rs.standard_normal(25)
    xs = np.linalg.solve(M, b)
    errs = []
    x, info = pcgmod.pcg(lambda v: M @ v, b, tol_abs=1e-11, max_iter=500,
                         callback=lambda it, xk, rk: errs.append((xk - xs) @ M @ (xk - xs)))
    assert all(e2 <= e1 * (1 + 1e-9) + 1e-24 for e1, e2 in zip(errs, errs[1:]))
    np.testing.assert_allclose(x, xs, rtol=1e-7, atol=1e-9)


# ------------------------------------------------------------------ IP-PMM pieces
def test_stepsize_spec_example():
    # x=(1,1), dx=(-2,-0.5) -> 0.995*min(1, 0.5, 2) = 0.4975 ; empty set -> 0.995 (A16)
    assert ippmm.stepsize(np.array([1.0, 1.0]), np.array([-2.0, -0.5])) == pytest.approx(0.4975, abs=1e-15)
    assert ippmm.stepsize(np.array([1.0, 1.0]), np.array([2.0, 0.5])) == 0.995


def test_duality_measure():
    # P:888 with J empty; S:321 x=z=(1,1) -> 1
    assert ippmm.duality_measure(np.ones(2), np.ones(2)) == 1.0
    assert ippmm.duality_measure(np.array([2.0, 4.0]), np.array([3.0, 0.5])) == 4.0


def test_newton_direction_block_structure_prop31():
    # Prop. 3.1: with dx, dz from the closed forms, blocks 1 and 3 of the Newton
    # system hold to rounding; block 2's residual equals the normal-eq residual.
    inst = make_config(0)
    rs = np.random.default_rng(13)
    n, m = inst.n, inst.m
    x = rs.uniform(0.1, 2, n)
    z = rs.uniform(0.1, 2, n)
    y = rs.standard_normal(m)
    rho, delta = 0.3, 0.07
    d = linops.scaling_d(inst.q, x, z, rho)
    r_d = inst.c + inst.q * x - inst.A.T @ y - z + rho * (x - x[::-1])
    r_p = inst.b - inst.A @ x - delta * (y - y[::-1])
    r_xz = -x * z
    holder = {}

    def solve_loose(xi):  # deliberately inexact: a few CG steps only
        sol, info = pcgmod.pcg(lambda v: linops.normal_matvec(inst.A, d, v, delta), xi,
                               tol_abs=0.0, max_iter=3)
        holder["theta"] = linops.normal_matvec(inst.A, d, sol, delta) - xi
        return sol, info

    dx, dy, dz, xi, _ = ippmm.newton_direction(inst.A, d, x, z, r_d, r_p, r_xz, solve_loose)
    b1, b2, b3 = ippmm.newton_block_residuals(inst.A, inst.q, rho, delta, x, z, dx, dy, dz, r_d, r_p, r_xz)
    scale = np.linalg.norm(r_d) + np.linalg.norm(inst.A.T @ dy) + np.linalg.norm(dz)
    assert np.linalg.norm(b1) <= 1e-13 * scale
    assert np.linalg.norm(b3) <= 1e-13 * (np.linalg.norm(r_xz) + np.linalg.norm(z * dx))
    assert np.linalg.norm(holder["theta"]) > 1e-6                 # the solve really was inexact
    np.testing.assert_allclose(b2, holder["theta"], rtol=1e-9, atol=1e-12)


def test_initial_point_hand_computed_n1():
    # App. B.2 on min 1/2 x^2 s.t. x = 1, x >= 0 (A=[1], b=1, c=0, q=1):
    # x~ = 1/11, y~ = (1/11)(1/11) = 1/121, z~ = 0 - 1/121 + 1/11 = 10/121, both >= 0 so
    # delta_p = delta_d = 0, gamma = 10/1331, delta~_p = 0.5 gamma / (10/121) = 1/22,
    # delta~_d = 0.5 gamma / (1/11) = 5/121
    A = np.array([[1.0]])
    solve = lambda r: (r / 11.0, {"iters": 0})  # noqa: E731 (AA^T + 10 I = 11)
    x0, y0, z0, _ = ippmm.initial_point(A, np.array([1.0]), np.array([1.0]), np.array([0.0]), solve)
    assert x0[0] == pytest.approx(1 / 11 + 1 / 22, rel=1e-15)
    assert y0[0] == pytest.approx(1 / 121, rel=1e-15)
    assert z0[0] == pytest.approx(10 / 121 + 5 / 121, rel=1e-15)


def _read_peu_rows():
    rows = []
    with open(os.path.join(GOLDEN, "peu_tables_5_6.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            p, k, r0, d0, r1, d1 = line.split()
            rows.append((p, int(k), float(r0), float(d0), float(r1), float(d1)))
    return rows


def test_peu_rule_form_matches_tables_5_6():
    # Tables 5-6: in rows where rho and delta shrink differently, the smaller
    # factor is (1 - r) (improved) and the larger is (1 - 2/3 r) (not improved), SURVEY A12.
    rows = _read_peu_rows()
    checked = 0
    for p, k, r0, d0, r1, d1 in rows:
        f_r, f_d = r1 / r0, d1 / d0
        if abs(f_r - f_d) <= 0.01 * max(f_r, f_d):
            # equal factors: both improved (or both not) with the same r
            assert ippmm.peu_factor(True, 1 - f_d) == pytest.approx(f_r, rel=0.02)
            continue
        small, large = min(f_r, f_d), max(f_r, f_d)
        r = 1.0 - small
        assert ippmm.peu_factor(True, r) == pytest.approx(small, rel=1e-12)
        assert ippmm.peu_factor(False, r) == pytest.approx(large, rel=0.03), (p, k)
        checked += 1
    assert checked >= 10


def test_peu_floor_value():
    # Tables 5-6 floor 5.00e-10
    assert ippmm.Options().reg_floor == 5e-10


# ------------------------------------------------------------------ end to end
def test_hand_kkt_n1_solution():
    # min 1/2 x^2, x = 1, x >= 0 -> x* = 1, y* = 1, z* = 0
    r = ippmm.solve(np.array([[1.0]]), np.array([1.0]), np.array([1.0]), np.array([0.0]),
                    ippmm.Options(path="krylov", ell=1))
    assert r.status == "optimal"
    assert r.x[0] == pytest.approx(1.0, abs=1e-7)
    assert r.y[0] == pytest.approx(1.0, abs=1e-6)
    assert r.z[0] == pytest.approx(0.0, abs=1e-7)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("path,ell", [("direct", 0), ("krylov", 2), ("krylov", 0)])
def test_tiny_qp_matches_active_set_enumeration(seed, path, ell):
    # S:425 / S:535-543: random tiny separable QPs vs brute-force active-set enumeration
    rs = np.random.default_rng(100 + seed)
    m, n = 3, 8
    A = rs.standard_normal((m, n))
    x0 = rs.uniform(0.2, 1.5, n)
    x0[rs.permutation(n)[:3]] = 0.0
    b = A @ x0
    q = rs.uniform(0.1, 2.0, n)           # Q > 0: unique x*
    c = rs.standard_normal(n)
    ref = enumerate_active_sets(A, q, b, c)
    r = ippmm.solve(A, q, b, c, ippmm.Options(path=path, ell=ell))
    assert r.status == "optimal"
    assert abs(r.obj - ref["obj"]) <= 1e-6 * max(1.0, abs(ref["obj"]))
    np.testing.assert_allclose(r.x, ref["x"], atol=1e-5)


def test_config0_direct_and_krylov_agree_and_bracket():
    inst = make_config(0)
    lo = inst.b @ inst.y0 - 0.5 * inst.x0 @ (inst.q * inst.x0)     # dual objective of (x0, y0, z0)
    hi = 0.5 * inst.x0 @ (inst.q * inst.x0) + inst.c @ inst.x0      # primal objective of x0
    rd = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="direct"))
    rk = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell))
    for r in (rd, rk):
        assert r.status == "optimal"
        assert lo - 1e-9 <= r.obj <= hi + 1e-9
        assert r.rel_p <= 1e-8 and r.rel_d <= 1e-8 and r.mu <= 1e-8
        assert abs(r.obj - r.dual_obj) <= 1e-6 * (1 + abs(r.obj))
    assert abs(rd.obj - rk.obj) <= 1e-7 * abs(rd.obj)


# ------------------------------------------------------------------ Philox
def test_philox_known_answer_vectors():
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            h = [int(t, 16) for t in line.split()]
            out = rng.philox4x32_10([h[0]], [h[1]], [h[2]], [h[3]], h[4], h[5])
            assert [int(o[0]) for o in out] == h[6:10]


def test_gaussian_omega_moments_and_layout():
    Om = rng.gaussian_omega(2000, 40, seed=5, stream=3)
    assert Om.shape == (2000, 40) and Om.flags["F_CONTIGUOUS"]
    assert abs(Om.mean()) < 0.01 and abs(Om.std() - 1) < 0.01
    # different streams / seeds are different matrices; same args reproduce bit-for-bit
    assert not np.array_equal(Om, rng.gaussian_omega(2000, 40, seed=5, stream=4))
    assert np.array_equal(Om, rng.gaussian_omega(2000, 40, seed=5, stream=3))
    # column-major linear index: a taller matrix has the first column's prefix as prefix
    Om2 = rng.gaussian_omega(2000, 41, seed=5, stream=3)
    np.testing.assert_array_equal(Om2[:, :40], Om)


def test_svm_instance_structure():
    # BASELINE configs[2] / SURVEY A23: A = [Xt, -Xt, I, -I], Xt = diag(y) X, b = 1, Q = diag(1 on w, 0 on xi, s)
    from synth.configs import svm_dense_A
    inst = make_config(2, m=40, n=6, ell=5)
    A = svm_dense_A(inst)
    N, d = 40, 6
    assert A.shape == (N, 2 * d + 2 * N) and inst.n == 2 * d + 2 * N
    Xt = inst.extra["Xt"]
    np.testing.assert_array_equal(A[:, :d], Xt)
    np.testing.assert_array_equal(A[:, d:2 * d], -Xt)
    np.testing.assert_array_equal(A[:, 2 * d:2 * d + N], np.eye(N))
    np.testing.assert_array_equal(A[:, 2 * d + N:], -np.eye(N))
    yl = inst.extra["labels"]
    # rows of diag(y) X are y_i (0.5 y_i 1 + g_i): mean of y_i * row over features is ~0.5
    assert abs(np.mean(Xt) - 0.5) < 0.2
    assert set(np.unique(yl)) <= {-1.0, 1.0}
    np.testing.assert_array_equal(inst.b, np.ones(N))
    np.testing.assert_array_equal(inst.q, np.r_[np.ones(2 * d), np.zeros(2 * N)])


def test_svm_tiny_qp_against_active_set():
    # the structured SVM QP solved by the oracle equals brute force on a tiny instance
    from synth.configs import svm_dense_A
    inst = make_config(2, m=4, n=2, ell=2)
    A = svm_dense_A(inst)
    ref = enumerate_active_sets(A, inst.q, inst.b, inst.c)
    r = ippmm.solve(A, inst.q, inst.b, inst.c, ippmm.Options(path="direct"))
    assert r.status == "optimal"
    assert abs(r.obj - ref["obj"]) <= 1e-6 * max(1.0, abs(ref["obj"]))


# ------------------------------------------------------------------ f3: preconditioner reuse
def test_prec_reuse_schedule_and_kkt():
    """prec_refresh = k rebuilds the Nystrom factors at outer iterations 0, k, 2k, ... (between
    rebuilds only mu_prec = delta_k changes); the solve still reaches the paper's tolerance (the
    Newton systems are solved to the same A8' tolerance whatever the preconditioner)."""
    inst = make_config(0)
    base = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=inst.ell))
    for k in (2, 3, 5):
        r = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=inst.ell, prec_refresh=k))
        assert r.status == "optimal" and r.rel_p <= 1e-8 and r.rel_d <= 1e-8 and r.mu <= 1e-8
        built = [l["k"] for l in r.log if l["prec_built"]]
        assert built == list(range(0, len(r.log), k))
        assert abs(r.obj - base.obj) <= abs(r.obj - r.dual_obj) + abs(base.obj - base.dual_obj) + 1e-7
    r1 = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=inst.ell, prec_refresh=1))
    assert r1.obj == base.obj and r1.inner_total == base.inner_total and all(l["prec_built"] for l in r1.log)


def test_prec_reuse_growth_trigger():
    """prec_growth: with an unbounded refresh period, rebuilds happen exactly when the previous
    iteration's PCG count exceeds growth x the count right after the last rebuild."""
    inst = make_config(0)
    g = 1.5
    r = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=inst.ell, prec_refresh=10 ** 6, prec_growth=g))
    assert r.status == "optimal"
    base = None
    for i, l in enumerate(r.log):
        if i == 0:
            assert l["prec_built"]
        else:
            prev = r.log[i - 1]["pcg_pred"] + r.log[i - 1]["pcg_corr"]
            assert l["prec_built"] == (prev > g * base)
        if l["prec_built"]:
            base = l["pcg_pred"] + l["pcg_corr"]


# ------------------------------------------------------------------ f2: partial Cholesky
def _chol_case(seed=0, m=12, n=40, delta=0.3):
    rs = np.random.default_rng(seed)
    A = rs.standard_normal((m, n))
    d = rs.uniform(0.05, 3.0, n)
    Nd = linops.dense_normal_matrix(A, d, delta)
    return A, d, delta, Nd


def test_partial_chol_diag_is_the_normal_diagonal():
    from oracle import partial_chol as pc
    A, d, delta, Nd = _chol_case()
    np.testing.assert_allclose(pc.diag_normal(A, d, delta), np.diag(Nd), rtol=1e-13)
    # pivots: the ell largest diagonal entries, ties -> smaller index (reading C1)
    assert list(pc.pivots(np.array([1.0, 3.0, 2.0, 3.0]), 2)) == [1, 3]


def test_partial_chol_full_rank_is_exact_and_zero_rank_is_jacobi():
    """ell = m: P_Chol = N_delta (S is empty); ell = 0: P_Chol = diag(N_delta) (eq. P:293-306)."""
    from oracle import partial_chol as pc
    A, d, delta, Nd = _chol_case(1)
    m = Nd.shape[0]
    F = pc.partial_cholesky(A, d, delta, m)
    np.testing.assert_allclose(pc.chol_precond_dense(F, m), Nd, rtol=1e-12, atol=1e-12 * np.abs(Nd).max())
    F0 = pc.partial_cholesky(A, d, delta, 0)
    np.testing.assert_allclose(pc.chol_precond_dense(F0, m), np.diag(np.diag(Nd)), rtol=1e-13)


def test_partial_chol_block_structure_schur_diagonal_and_inverse():
    """P_Chol equals N_delta on the pivot rows/columns, its complement block is L21 L21^T + diag(S),
    diag(S) is the diagonal of the exact Schur complement, and the closed-form inverse
    inverts it."""
    from oracle import partial_chol as pc
    A, d, delta, Nd = _chol_case(2, m=15, n=50)
    m, ell = Nd.shape[0], 5
    F = pc.partial_cholesky(A, d, delta, ell)
    Pm = pc.chol_precond_dense(F, m)
    P, Q = F["P"], F["Q"]
    np.testing.assert_allclose(Pm[P, :], Nd[P, :], rtol=1e-12, atol=1e-12 * np.abs(Nd).max())
    S = Nd[np.ix_(Q, Q)] - Nd[np.ix_(Q, P)] @ np.linalg.solve(Nd[np.ix_(P, P)], Nd[np.ix_(P, Q)])
    np.testing.assert_allclose(F["dS"], np.diag(S), rtol=1e-11)
    assert np.all(np.diag(Nd)[P].min() >= np.diag(Nd)[Q].max())     # the ell largest diagonal entries
    rs = np.random.default_rng(3)
    for _ in range(3):
        v = rs.standard_normal(m)
        np.testing.assert_allclose(Pm @ pc.chol_precond_inv_apply(F, v), v, rtol=1e-10, atol=1e-10)


def test_partial_chol_pcg_full_rank_one_iteration():
    from oracle import partial_chol as pc
    A, d, delta, Nd = _chol_case(4)
    m = Nd.shape[0]
    F = pc.partial_cholesky(A, d, delta, m)
    b = np.random.default_rng(5).standard_normal(m)
    x, info = pcgmod.pcg(lambda v: Nd @ v, b, lambda v: pc.chol_precond_inv_apply(F, v), tol_abs=1e-10 * np.linalg.norm(b))
    assert info["iters"] <= 1
    np.testing.assert_allclose(Nd @ x, b, rtol=1e-9, atol=1e-9)


def test_chol_ippmm_tiny_qps_match_brute_force():
    """Chol-IP-PMM (precond="chol") reaches the brute-force active-set optimum of tiny QPs."""
    rs = np.random.default_rng(11)
    for t in range(3):
        m, n = 3, 9
        A = rs.standard_normal((m, n))
        x0 = rs.uniform(0.5, 1.5, n)
        q = rs.uniform(0.1, 1.0, n)
        b = A @ x0
        c = A.T @ rs.standard_normal(m) + rs.uniform(-0.5, 1.5, n) - q * x0
        bf = enumerate_active_sets(A, q, b, c)
        f_bf, x_bf = bf["obj"], bf["x"]
        r = ippmm.solve(A, q, b, c, ippmm.Options(ell=2, precond="chol"))
        assert r.status == "optimal"
        assert abs(r.obj - f_bf) <= 1e-6 * max(1.0, abs(f_bf))
        assert np.abs(r.x - x_bf).max() <= 1e-5


# ------------------------------------------------------------------ f1: free and box variables
def _gen_qp(rs, m, n, vtype, ub_scale=1.0):
    A = rs.standard_normal((m, n))
    vt = np.asarray(vtype)
    x0 = rs.uniform(0.2, 0.8, n) * ub_scale
    x0[vt == 1] = rs.standard_normal(int((vt == 1).sum()))
    u = np.where(vt == 2, ub_scale, 0.0)
    q = rs.uniform(0.1, 1.0, n)
    b = A @ x0
    c = rs.standard_normal(n)
    return A, q, b, c, u


def test_general_form_all_nonnegative_reduces_to_standard():
    """vtype = all I (u = 0, w = s = 0): the general-form iteration is the standard one."""
    from oracle import ippmm_gen
    inst = make_config(0)
    r0 = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=inst.ell))
    rg = ippmm_gen.solve_general(inst.A, inst.q, inst.b, inst.c, np.zeros(inst.n, dtype=int), np.zeros(inst.n),
                                 ippmm.Options(ell=inst.ell))
    # identical formulas; only the rounding of the residual norms (sqrt of sums vs np.linalg.norm)
    # differs, which moves the PCG stopping points by a few iterations
    assert rg.status == "optimal" and rg.outer == r0.outer
    assert abs(rg.inner_total - r0.inner_total) <= 0.01 * r0.inner_total
    assert abs(rg.obj - r0.obj) <= 1e-9 * abs(r0.obj)


@pytest.mark.parametrize("seed", range(4))
def test_general_form_tiny_qps_match_brute_force(seed):
    """Free / non-negative / box variables mixed: the solve reaches the brute-force optimum."""
    from oracle import ippmm_gen
    from oracle.active_set import enumerate_active_sets_general
    rs = np.random.default_rng(100 + seed)
    vtype = [0, 0, 1, 2, 2, 2, 0, 2]
    A, q, b, c, u = _gen_qp(rs, 3, len(vtype), vtype)
    bf = enumerate_active_sets_general(A, q, b, c, np.array(vtype), u)
    for path in ("direct", "krylov"):
        r = ippmm_gen.solve_general(A, q, b, c, vtype, u, ippmm.Options(path=path, ell=2))
        assert r.status == "optimal"
        assert abs(r.obj - bf["obj"]) <= 1e-6 * max(1.0, abs(bf["obj"]))
        assert np.abs(r.x - bf["x"]).max() <= 1e-5
        vt = np.array(vtype)
        assert np.all(r.x[vt != 1] > 0) and np.all(r.x[vt == 2] < u[vt == 2])       # strictly interior iterates
        assert np.allclose(r.w[vt == 2], u[vt == 2] - r.x[vt == 2], atol=1e-7)


def test_free_variables_equal_the_split_formulation():
    """x_F free is equivalent to x_F = x+ - x- with x+, x- >= 0: same optimal objective."""
    from oracle import ippmm_gen
    rs = np.random.default_rng(7)
    m, n = 4, 10
    vtype = np.array([1, 1, 0, 0, 0, 0, 0, 0, 1, 0])
    A, q, b, c, u = _gen_qp(rs, m, n, vtype)
    q[vtype == 1] = 0.5
    rg = ippmm_gen.solve_general(A, q, b, c, vtype, u, ippmm.Options(path="direct"))
    F = np.where(vtype == 1)[0]
    As = np.hstack([A, -A[:, F]])
    qs = np.concatenate([q, q[F]])
    cs = np.concatenate([c, -c[F]])
    # with Q: 1/2 q (x+ - x-)^2 != 1/2 q (x+^2 + x-^2) in general -> compare on q_F -> the split optimum
    # has x+ x- = 0, where both coincide
    rs_ = ippmm.solve(As, qs, b, cs, ippmm.Options(path="direct"))
    assert rg.status == "optimal" and rs_.status == "optimal"
    assert abs(rg.obj - rs_.obj) <= 1e-6 * max(1.0, abs(rs_.obj))


# ------------------------------------------------------------------ f3: adaptive rank (reading F1)
def test_adaptive_rank_off_is_the_fixed_rank_solve():
    inst = make_config(1, m=120, n=480, ell=8)
    r0 = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=8))
    r1 = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=8, ell_max=8))
    assert r0.outer == r1.outer and r0.inner_total == r1.inner_total and r0.obj == r1.obj
    assert all(l["ell"] == 8 for l in r1.log)


def test_adaptive_rank_follows_the_doubling_rule():
    """F1: the rank doubles (capped) for the next build exactly when lam_hat_ell > tau * delta_k after a
    build; never shrinks; the rank-40 spike of config 1 is captured and PCG work drops."""
    inst = make_config(1, m=200, n=800, ell=10)
    tau, cap = 10.0, 80
    r = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=10, ell_max=cap, ell_tau=tau))
    rf = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(ell=10))
    assert r.status == "optimal" and rf.status == "optimal"
    ells = [l["ell"] for l in r.log]
    assert ells[0] == 10 and all(b >= a for a, b in zip(ells, ells[1:]))
    for a, b in zip(r.log, r.log[1:]):
        grow = a["prec_built"] and a["lam_ell"] > tau * a["delta"] and a["ell"] < cap
        assert b["ell"] == (min(2 * a["ell"], cap) if grow else a["ell"])
    assert max(ells) == cap                                   # the spike (rank 40) needs > 40
    assert r.inner_total < 0.5 * rf.inner_total
    assert abs(r.obj - rf.obj) <= 1e-6 * abs(rf.obj)


def test_general_form_elementwise_pieces_by_hand():
    """Theta^{-1}, mu and the two-set step length of (P~)/(D~) on a hand-worked 3-variable example
    (one variable in each of I, F, J; P:1431 elimination)."""
    from oracle import ippmm_gen
    vt = np.array([0, 1, 2])
    x = np.array([2.0, -3.0, 0.5])
    z = np.array([4.0, 0.0, 1.0])
    w = np.array([0.0, 0.0, 1.5])
    s = np.array([0.0, 0.0, 3.0])
    th = ippmm_gen.theta_inv(x, z, w, s, vt)
    assert np.allclose(th, [4.0 / 2.0, 0.0, 1.0 / 0.5 + 3.0 / 1.5])
    # mu = (x_IJ^T z_IJ + w_J^T s_J) / (|IJ| + |J|) = (8 + 0.5 + 4.5) / 3
    assert abs(ippmm_gen.mu_general(x, z, w, s, vt) - 13.0 / 3.0) < 1e-15
    # step: x_I blocks at 2/4 = 0.5, x_J at 0.5/1 = 0.5, w_J at 1.5/0.5 = 3; the free x is ignored
    dx = np.array([-4.0, -100.0, -1.0])
    dw = np.array([0.0, 0.0, -0.5])
    assert abs(ippmm_gen.stepsize_general(x, dx, w, dw, vt) - 0.995 * 0.5) < 1e-15
    dw2 = np.array([0.0, 0.0, -6.0])    # now w blocks first: 1.5 / 6 = 0.25
    assert abs(ippmm_gen.stepsize_general(x, dx, w, dw2, vt) - 0.995 * 0.25) < 1e-15


def test_general_newton_direction_solves_the_linearised_system():
    """With an exact normal-equation solve, Alg. 4's direction satisfies every block row of the
    Newton system P:1431 (the 5 x 5 block system in dx, dy, dw, dz, ds) to rounding."""
    from oracle import ippmm_gen
    rs = np.random.default_rng(5)
    m, n = 4, 9
    vt = np.array([0, 1, 2, 0, 2, 1, 0, 2, 2])
    I, F, J, IJ = ippmm_gen.masks(vt)
    A = rs.standard_normal((m, n))
    q = rs.uniform(0.1, 1.0, n)
    x = np.where(F, rs.standard_normal(n), rs.uniform(0.2, 1.0, n))
    z = np.where(F, 0.0, rs.uniform(0.2, 1.0, n))
    w = np.where(J, rs.uniform(0.2, 1.0, n), 0.0)
    s = np.where(J, rs.uniform(0.2, 1.0, n), 0.0)
    rho, delta = 0.3, 0.2
    d = 1.0 / (q + ippmm_gen.theta_inv(x, z, w, s, vt) + rho)
    r_d, r_p = rs.standard_normal(n), rs.standard_normal(m)
    r_u = np.where(J, rs.standard_normal(n), 0.0)
    r_xz = np.where(IJ, rs.standard_normal(n), 0.0)
    r_ws = np.where(J, rs.standard_normal(n), 0.0)
    N = (A * d) @ A.T + delta * np.eye(m)
    solve = lambda xi: (np.linalg.solve(N, xi), {})  # noqa: E731
    dx, dy, dz, dw, ds, _ = ippmm_gen.newton_direction_general(A, d, x, z, w, s, vt, r_d, r_p, r_u, r_xz, r_ws, solve)
    # row 1: -(Q + rho I) dx + A^T dy + dz - ds = r_d   (sign convention of Alg. 4 / reading G0)
    assert np.allclose(-(q + rho) * dx + A.T @ dy + dz - ds, r_d, atol=1e-10)
    assert np.allclose(A @ dx + delta * dy, r_p, atol=1e-10)                           # row 2
    assert np.allclose((dx + dw)[J], r_u[J], atol=1e-12)                                 # row 3
    assert np.allclose((z * dx + x * dz)[IJ], r_xz[IJ], atol=1e-12)                      # row 4
    assert np.allclose((s * dw + w * ds)[J], r_ws[J], atol=1e-12)                        # row 5
    assert np.all(dz[F] == 0) and np.all(dw[~J] == 0) and np.all(ds[~J] == 0)


def test_general_form_all_free_is_the_kkt_solution():
    """Every variable free (reading G5): min 1/2 x^T Q x + c^T x s.t. A x = b has the closed-form KKT
    solution [Q A^T; A 0] [x; -y] = [-c; b]; the general-form solve reaches it (both paths)."""
    from oracle import ippmm_gen
    rs = np.random.default_rng(9)
    m, n = 3, 7
    A = rs.standard_normal((m, n))
    q = rs.uniform(0.5, 2.0, n)
    b = rs.standard_normal(m)
    c = rs.standard_normal(n)
    K = np.block([[np.diag(q), A.T], [A, np.zeros((m, m))]])
    sol = np.linalg.solve(K, np.concatenate([-c, b]))
    x_kkt, y_kkt = sol[:n], -sol[n:]
    vt = np.ones(n, dtype=int)
    for path in ("direct", "krylov"):
        r = ippmm_gen.solve_general(A, q, b, c, vt, np.zeros(n), ippmm.Options(path=path, ell=2))
        assert r.status == "optimal"
        assert np.abs(r.x - x_kkt).max() <= 1e-7 and np.abs(r.y - y_kkt).max() <= 1e-7
        assert np.all(r.z == 0)


# ------------------------------------------------------------------ App. B.2 initial point with shifts (round 2)
def test_initial_point_shift_branch_hand_computed():
    """App. B.2 with both shifts active and different (delta_p != delta_d > 0), so the
    -1.5 min shifts, gamma and the delta~_d denominator reading A13
    (sum(x~ + delta_p), P:1473 prints sum(x~ + delta_d)) are all exercised.
    Worked by hand: A = [1 2], q = 0, b = -3, c = (1, -2); A A^T + 10 I = 15.
      x~ = A^T (-3/15) = (-0.2, -0.4);  A (c + Q x~) = 1 - 4 = -3 -> y~ = -0.2
      z~ = c - A^T y~ = (1.2, -1.6)
      delta_p = -1.5 (-0.4) = 0.6,  delta_d = -1.5 (-1.6) = 2.4
      x~ + delta_p = (0.4, 0.2),  z~ + delta_d = (3.6, 0.8),  gamma = 1.44 + 0.16 = 1.6
      delta~_p = 0.6 + 0.8 / 4.4 = 0.6 + 2/11
      delta~_d = 2.4 + 0.8 / 0.6 = 2.4 + 4/3   (printed denominator sum(x~ + delta_d) = 4.2 would give 2.4 + 4/21)
    """
    A = np.array([[1.0, 2.0]])
    solve = lambda r: (r / 15.0, {"iters": 0})  # noqa: E731
    x0, y0, z0, _ = ippmm.initial_point(A, np.zeros(2), np.array([-3.0]), np.array([1.0, -2.0]), solve)
    dpt, ddt = 0.6 + 2.0 / 11.0, 2.4 + 4.0 / 3.0
    np.testing.assert_allclose(x0, [-0.2 + dpt, -0.4 + dpt], rtol=1e-14)
    np.testing.assert_allclose(y0, [-0.2], rtol=1e-14)
    np.testing.assert_allclose(z0, [1.2 + ddt, -1.6 + ddt], rtol=1e-14)
    # the alternative readings differ well above rounding: the pin can tell them apart
    assert abs(z0[0] - (1.2 + 2.4 + 4.0 / 21.0)) > 1.0           # printed P:1473 denominator
    assert abs(x0[0] - (-0.2 + 0.4 + 1.6 / 2.0 / (1.2 + 1.6 + 1.6 * 2 / 3 * 2))) > 0.05   # shift factor 1, not 1.5


def test_initial_point_with_q_term_hand_computed():
    """Same construction with Q != 0 (the Q x~ terms of y~ and z~):
    A = [1 2], q = (1, 0), b = -3, c = (1, -2), A A^T + 10 I = 15.
      x~ = (-0.2, -0.4);  c + Q x~ = (0.8, -2);  A(c + Q x~) = -3.2 -> y~ = -16/75
      z~ = c - A^T y~ + Q x~ = (1 + 16/75 - 0.2, -2 + 32/75) = (76/75, -118/75)
      delta_p = 0.6, delta_d = 1.5 * 118/75 = 2.36
      x~ + delta_p = (0.4, 0.2), z~ + delta_d = (76/75 + 2.36, -118/75 + 2.36) = (253/75, 59/75)
      gamma = 0.4 * 253/75 + 0.2 * 59/75 = 113/75;  sum(z~ + delta_d) = 312/75;  sum(x~ + delta_p) = 0.6
      delta~_p = 0.6 + (113/150) / (312/75) = 0.6 + 113/624;  delta~_d = 2.36 + (113/150) / 0.6 = 2.36 + 113/90"""
    A = np.array([[1.0, 2.0]])
    solve = lambda r: (r / 15.0, {"iters": 0})  # noqa: E731
    x0, y0, z0, _ = ippmm.initial_point(A, np.array([1.0, 0.0]), np.array([-3.0]), np.array([1.0, -2.0]), solve)
    F = Fraction
    dpt = F(3, 5) + F(113, 624)
    ddt = F(236, 100) + F(113, 90)
    np.testing.assert_allclose(x0, [float(F(-1, 5) + dpt), float(F(-2, 5) + dpt)], rtol=1e-14)
    np.testing.assert_allclose(y0, [float(F(-16, 75))], rtol=1e-14)
    np.testing.assert_allclose(z0, [float(F(76, 75) + ddt), float(F(-118, 75) + ddt)], rtol=1e-14)


def test_general_initial_point_shift_branch_hand_computed():
    """App. B.2 general form with I, J (box) and F (free) variables; readings G2 (delta~_d
    denominator sum(x~_IJ + delta_p) + sum(w~_J + delta_p)) and G3 (A A^T + 10 I, x~_F not shifted).
    Worked by hand: A = [1 2 1], vtype = (I, J, F), u = (0, 1, 0), q = 0, b = -3.8, c = (1, -2, 0.5);
    A A^T + 10 I = 16.
      x~ = u/2 + A^T (b - A u / 2)/16 = (0, 0.5, 0) + (-4.8/16) (1, 2, 1) = (-0.3, -0.1, -0.3)
      y~ = A c / 16 = -2.5/16 = -0.15625;  g = c - A^T y~ = (1.15625, -1.6875, 0.65625)
      z~ = (g_I, g_J / 2, 0) = (1.15625, -0.84375, 0);  s~_J = 0.84375;  w~_J = u_J - x~_J = 1.1
      delta_p = max(-1.5 min(-0.3, -0.1), -1.5 (1.1), 0) = 0.45
      delta_d = max(-1.5 min(1.15625, -0.84375), -1.5 (0.84375), 0) = 1.265625
      gamma_xz = (0.15, 0.35).(2.421875, 0.421875) = 0.5109375
      gamma_ws = (1.1 + 0.45)(0.84375 + 1.265625) = 3.26953125;  gamma = 3.78046875
      den_p = 2.421875 + 0.421875 + 2.109375 = 4.953125;  den_d = 0.15 + 0.35 + 1.55 = 2.05
      delta~_p = 0.45 + 1.890234375 / 4.953125;  delta~_d = 1.265625 + 1.890234375 / 2.05
      x0 = (x~_I + delta~_p, x~_J + delta~_p, x~_F),  w0_J = 1.1 + delta~_p,
      z0 = (z~_I + delta~_d, z~_J + delta~_d, 0),  s0_J = 0.84375 + delta~_d"""
    from oracle import ippmm_gen
    A = np.array([[1.0, 2.0, 1.0]])
    solve = lambda r: (r / 16.0, {"iters": 0})  # noqa: E731
    vtype = np.array([0, 2, 1], np.int8)
    u = np.array([0.0, 1.0, 0.0])
    x0, y0, z0, w0, s0 = ippmm_gen.initial_point_general(A, np.zeros(3), np.array([-3.8]),
                                                         np.array([1.0, -2.0, 0.5]), vtype, u, solve)
    dpt = 0.45 + 1.890234375 / 4.953125
    ddt = 1.265625 + 1.890234375 / 2.05
    np.testing.assert_allclose(x0, [-0.3 + dpt, -0.1 + dpt, -0.3], rtol=1e-14)
    np.testing.assert_allclose(y0, [-0.15625], rtol=1e-14)
    np.testing.assert_allclose(z0, [1.15625 + ddt, -0.84375 + ddt, 0.0], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(w0, [0.0, 1.1 + dpt, 0.0], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(s0, [0.0, 0.84375 + ddt, 0.0], rtol=1e-14, atol=1e-15)
    # printed P:1473 denominators (x~ + delta_d, w~ + delta_d) give a different delta~_d
    printed = 1.265625 + 1.890234375 / ((-0.3 + 1.265625) + (-0.1 + 1.265625) + (1.1 + 1.265625))
    assert abs(ddt - printed) > 0.3


# ------------------------------------------------------------------ exact f* by dual semismooth Newton (§8(c) P9)
@pytest.mark.parametrize("seed", range(5))
def test_ssn_matches_active_set_enumeration(seed):
    from oracle import ssn
    rs = np.random.default_rng(300 + seed)
    m, n = 3, 9
    A = rs.standard_normal((m, n))
    x0 = rs.uniform(0.2, 1.5, n)
    x0[rs.permutation(n)[:4]] = 0.0
    b = A @ x0
    q = rs.uniform(0.1, 2.0, n)
    c = rs.standard_normal(n)
    ref = enumerate_active_sets(A, q, b, c)
    r = ssn.solve(A, q, b, c)
    assert abs(r["obj"] - ref["obj"]) <= 1e-10 * max(1.0, abs(ref["obj"]))
    np.testing.assert_allclose(r["x"], ref["x"], atol=1e-9)


def test_ssn_exact_kkt_and_strong_duality_config3_full():
    """SSN's point satisfies x >= 0, z >= 0 and x o z = 0 exactly (by construction of x(y)), the primal
    residual is at rounding level and the primal and dual objectives coincide (strong duality, Q > 0)."""
    from oracle import ssn
    inst = make_config(3)
    r = ssn.solve(inst.A, inst.q, inst.b, inst.c)
    assert r["x"].min() >= 0 and r["z"].min() >= -1e-15 * np.abs(inst.c).max()
    assert np.max(np.abs(r["x"] * r["z"])) <= 1e-15
    assert r["rel_p"] <= 1e-10
    assert abs(r["obj"] - r["dual_obj"]) <= 1e-12 * (1 + abs(r["obj"]))


def _band(A, q, b, c, res):
    rP = b - A @ res.x
    rD = c + q * res.x - A.T @ res.y - res.z
    return abs(res.obj - res.dual_obj) + np.linalg.norm(res.x) * np.linalg.norm(rD) + np.linalg.norm(res.y) * np.linalg.norm(rP)


@pytest.mark.parametrize("idx,kw,path", [(3, {}, "krylov"), (1, dict(m=200, n=800, ell=20), "direct"),
                                         (1, dict(m=200, n=800, ell=20), "krylov")])
def test_ippmm_lands_within_its_certified_band_of_ssn_fstar(idx, kw, path):
    """The IP-PMM oracle's objective at the paper's tolerance (1e-8) is within its certified band
    (weak duality with residuals) of the EXACT f* from dual semismooth Newton — an
    independent method (no barrier, no Krylov solve).  Full-size config 3; reduced config 1 on both paths."""
    from oracle import ssn
    inst = make_config(idx, **kw)
    fstar = ssn.solve(inst.A, inst.q, inst.b, inst.c)
    assert fstar["rel_p"] <= 1e-10
    r = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path=path, ell=inst.ell))
    assert r.status == "optimal"
    band = _band(inst.A, inst.q, inst.b, inst.c, r)
    assert abs(r.obj - fstar["obj"]) <= band + 1e-12 * abs(fstar["obj"])
    # x* is unique (Q > 0, A19): the IP-PMM iterate is close to it
    assert np.linalg.norm(r.x - fstar["x"]) <= 1e-4 * np.linalg.norm(fstar["x"])


# ------------------------------------------------------------------ config 2 operator and Woodbury path D (A23)
def test_svm_operator_equals_the_materialised_A():
    from oracle import svm
    from synth.configs import svm_dense_A
    inst = make_config(2, m=60, n=7, ell=5)
    A = svm_dense_A(inst)
    op = svm.SvmOperator(inst.extra["Xt"])
    rs = np.random.default_rng(1)
    X = rs.standard_normal((inst.n, 3))
    Y = rs.standard_normal((inst.m, 3))
    assert op.shape == A.shape
    np.testing.assert_allclose(op @ X, A @ X, rtol=0, atol=1e-13)
    np.testing.assert_allclose(op.T @ Y, A.T @ Y, rtol=0, atol=1e-13)
    d = rs.uniform(0.1, 2.0, inst.n)
    np.testing.assert_allclose(op.dense_normal_matrix(d, 0.3), linops.dense_normal_matrix(A, d, 0.3), rtol=1e-13, atol=1e-12)


def test_woodbury_solve_equals_dense_solve():
    """The capacitance form is an exact identity: it matches a dense LU solve of A D A^T + delta I."""
    from oracle import svm
    from synth.configs import svm_dense_A
    inst = make_config(2, m=300, n=20, ell=10)
    A = svm_dense_A(inst)
    op = svm.SvmOperator(inst.extra["Xt"])
    rs = np.random.default_rng(2)
    for delta in (1e-8, 1e-3, 10.0):
        d = np.exp(rs.uniform(-12, 4, inst.n))                    # IPM-like spread of D
        r = rs.standard_normal(inst.m)
        sol = op.direct_solver(d, delta)(r)[0]
        M = linops.dense_normal_matrix(A, d, delta)
        ref = np.linalg.solve(M, r)
        # backward stable (residual at rounding of ||M|| ||sol||), forward error within kappa eps
        nM = np.linalg.norm(M, 2)
        assert np.linalg.norm(M @ sol - r) <= 1e-13 * (nM * np.linalg.norm(sol) + np.linalg.norm(r))
        assert np.linalg.norm(sol - ref) <= 1e-14 * np.linalg.cond(M) * np.linalg.norm(ref)


def test_svm_path_d_operator_agrees_with_dense_paths_and_brute_force():
    """Path D through the operator (Woodbury) = path D on the materialised A = path K (Nystrom PCG),
    and the tiny instance equals brute-force active-set enumeration."""
    from oracle import svm
    from synth.configs import svm_dense_A
    inst = make_config(2, m=300, n=20, ell=10)
    A = svm_dense_A(inst)
    op = svm.SvmOperator(inst.extra["Xt"])
    rw = ippmm.solve(op, inst.q, inst.b, inst.c, ippmm.Options(path="direct"))
    rd = ippmm.solve(A, inst.q, inst.b, inst.c, ippmm.Options(path="direct"))
    rk = ippmm.solve(A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=10))
    assert rw.status == rd.status == rk.status == "optimal"
    assert rw.outer == rd.outer
    assert abs(rw.obj - rd.obj) <= 1e-10 * abs(rd.obj)
    assert abs(rk.obj - rd.obj) <= _band(A, inst.q, inst.b, inst.c, rk) + _band(A, inst.q, inst.b, inst.c, rd)
    tiny = make_config(2, m=4, n=2, ell=2)
    ref = enumerate_active_sets(svm_dense_A(tiny), tiny.q, tiny.b, tiny.c)
    rt = ippmm.solve(svm.SvmOperator(tiny.extra["Xt"]), tiny.q, tiny.b, tiny.c, ippmm.Options(path="direct"))
    assert abs(rt.obj - ref["obj"]) <= 1e-6 * max(1.0, abs(ref["obj"]))
