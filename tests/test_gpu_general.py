"""GPU parity for free and box-constrained variables, problem (P~)/(D~) (Alg. 5 P:858-918,
App. B.2-B.3): the CUDA path (nys_ipppmm_solve with vtype / ub) against
oracle.ippmm_gen.solve_general on seeded mixed-type instances (synth.make_general)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ippmm, ippmm_gen  # noqa: E402
from synth import make_general  # noqa: E402

pytestmark = pytest.mark.gpu


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dtype).cuda()


def band_general(inst, x, y, z, s, p, d):
    """Weak duality with residuals for (P~)/(D~) (extends A17; G1): for any feasible x*,
    f(x*) >= d + r_D^T x*  (convexity of 1/2 x^T Q x, z^T x* >= 0 on IJ, -s^T x* >= -u^T s on J),
    and f* <= p + |y*^T r_P| + |s*^T r_U| (sensitivity to b and u).  So f* is determined to
    |p - d| + ||x|| ||r_D|| + ||y|| ||r_P|| + ||s|| ||r_U||."""
    vt, u = inst.extra["vtype"], inst.extra["ub"]
    J = vt == 2
    w = np.where(J, u - x, 0.0)
    rP = inst.b - inst.A @ x
    rD = inst.c + inst.q * x - inst.A.T @ y - z + s
    rU = np.where(J, u - x - w, 0.0)
    return (abs(p - d) + np.linalg.norm(x) * np.linalg.norm(rD) + np.linalg.norm(y) * np.linalg.norm(rP)
            + np.linalg.norm(s) * np.linalg.norm(rU))


def _ctx():
    from paper_2404_14524_b200 import Context
    return Context(0)


def _solve(ctx, inst, host=False, **kw):
    from paper_2404_14524_b200 import colmajor_device
    vt, u = inst.extra["vtype"], inst.extra["ub"]
    if host:
        lda = ((inst.m + 31) // 32) * 32                 # the layout colmajor_device uses
        Ah = np.zeros((inst.n, lda))
        Ah[:, :inst.m] = inst.A.T
        return ctx.nys_ipppmm_solve(Ah, lda, inst.m, inst.q, inst.b, inst.c, ell=inst.ell, host=True,
                                    vtype=vt, ub=u, **kw)
    Ad, lda = colmajor_device(inst.A)
    return ctx.nys_ipppmm_solve(Ad, lda, inst.m, dev(inst.q), dev(inst.b), dev(inst.c), ell=inst.ell,
                                vtype=dev(vt, torch.int8), ub=dev(u), **kw)


def _h(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


GEN_CASES = [(100, 300, 0.2, 0.3, 20), (200, 800, 0.1, 0.5, 20), (50, 400, 0.0, 1.0, 20), (80, 240, 1 / 3, 0.0, 20),
             (120, 600, 0.25, 0.25, 0), (257, 1031, 0.15, 0.35, 32)]


@pytest.mark.parametrize("m,n,ff,fb,ell", GEN_CASES)
def test_general_ipppmm_matches_oracle(m, n, ff, fb, ell):
    inst = make_general(m, n, ff, fb, ell=ell)
    vt, u = inst.extra["vtype"], inst.extra["ub"]
    I, F, J = vt == 0, vt == 1, vt == 2
    ref = ippmm_gen.solve_general(inst.A, inst.q, inst.b, inst.c, vt, u, ippmm.Options(path="krylov", ell=ell))
    assert ref.status == "optimal"
    ctx = _ctx()
    g = _solve(ctx, inst)
    torch.cuda.synchronize()
    x, y, z, w, s = (_h(g[k]) for k in ("x", "y", "z", "w", "s"))
    assert g["status"] == 0 and g["rel_p"] <= 1e-8 and g["rel_d"] <= 1e-8 and g["mu"] <= 1e-8
    # structure of the iterate: interior on I and J, z_F = 0, w, s zero off J
    assert np.all(x[I | J] > 0) and np.all(z[I | J] > 0) and np.all(z[F] == 0)
    assert np.all(w[J] > 0) and np.all(s[J] > 0) and np.all(w[~J] == 0) and np.all(s[~J] == 0)
    # G1 residuals recomputed here in fp64 from the returned iterate
    bn = np.sqrt(inst.b @ inst.b + u[J] @ u[J])
    rP = np.concatenate([inst.b - inst.A @ x, (u - x - w)[J]])
    rD = inst.c + inst.q * x - inst.A.T @ y - z + s
    assert np.linalg.norm(rP) / (1 + bn) <= 1.01e-8
    assert np.linalg.norm(rD) / (1 + np.linalg.norm(inst.c)) <= 1.01e-8
    mu = (x[I | J] @ z[I | J] + w[J] @ s[J]) / ((I | J).sum() + J.sum())
    assert abs(mu - g["mu"]) <= 1e-6 * g["mu"] + 1e-20
    f = 0.5 * x @ (inst.q * x) + inst.c @ x
    assert abs(f - g["obj"]) <= 1e-10 * max(1.0, abs(f))
    dual = inst.b @ y - u[J] @ s[J] - 0.5 * x @ (inst.q * x)
    assert abs(dual - g["dual_obj"]) <= 1e-10 * max(1.0, abs(dual))
    band_ = (band_general(inst, x, y, z, s, g["obj"], g["dual_obj"]) +
              band_general(inst, ref.x, ref.y, ref.z, ref.s, ref.obj, ref.dual_obj))
    tol = 1e-7 * max(1.0, abs(ref.obj))   # strict (north_star); the certified band is only reported
    print(f"obj diff vs oracle: strict tol {tol:.3e}, certified bands {band_:.3e}")
    print(f"gpu obj {g['obj']!r} ref {ref.obj!r} outer {g['outer']}/{ref.outer} inner {g['inner']}/{ref.inner_total}")
    assert abs(g["obj"] - ref.obj) <= tol
    assert abs(g["outer"] - ref.outer) <= 2
    # first iterations follow the oracle's trajectory (same initial point, same sketches)
    for k in range(min(2, len(g["log"]), len(ref.log))):
        assert abs(g["log"][k]["mu"] - ref.log[k]["mu"]) <= 1e-6 * ref.log[k]["mu"]
        assert abs(g["log"][k]["alpha_p"] - ref.log[k]["alpha_p"]) <= 1e-6
        assert abs(g["log"][k]["alpha_d"] - ref.log[k]["alpha_d"]) <= 1e-6
        assert (g["log"][k]["pcg_pred"], g["log"][k]["pcg_corr"]) == (ref.log[k]["pcg_pred"], ref.log[k]["pcg_corr"])
    ctx.close()


def test_general_host_pointers_match_device():
    inst = make_general(90, 350, 0.2, 0.4, ell=16, seed=11)
    ctx = _ctx()
    gd = _solve(ctx, inst)
    gh = _solve(ctx, inst, host=True)
    torch.cuda.synchronize()
    assert gd["status"] == 0 and gh["status"] == 0
    assert gd["outer"] == gh["outer"] and gd["inner"] == gh["inner"]
    for k in ("x", "y", "z", "w", "s"):
        assert np.array_equal(_h(gd[k]), gh[k])
    ctx.close()


def test_general_all_nonnegative_equals_standard_path():
    """vtype = 0 everywhere: the f1 kernels reproduce the (P)/(D) path."""
    from paper_2404_14524_b200 import colmajor_device
    from synth import make_config
    inst = make_config(1, m=200, n=800, ell=20)
    ctx = _ctx()
    Ad, lda = colmajor_device(inst.A)
    g0 = ctx.nys_ipppmm_solve(Ad, lda, inst.m, dev(inst.q), dev(inst.b), dev(inst.c), ell=inst.ell)
    g1 = ctx.nys_ipppmm_solve(Ad, lda, inst.m, dev(inst.q), dev(inst.b), dev(inst.c), ell=inst.ell,
                              vtype=torch.zeros(inst.n, dtype=torch.int8, device="cuda"))
    torch.cuda.synchronize()
    assert g0["status"] == 0 and g1["status"] == 0 and g0["outer"] == g1["outer"]
    assert abs(g0["inner"] - g1["inner"]) <= 0.01 * g0["inner"]
    assert abs(g0["obj"] - g1["obj"]) <= 1e-9 * abs(g0["obj"])
    assert np.all(_h(g1["w"]) == 0) and np.all(_h(g1["s"]) == 0)
    ctx.close()


def test_general_rejects_bad_vtype_and_bounds():
    from paper_2404_14524_b200 import NysError
    inst = make_general(40, 120, 0.2, 0.3, ell=8, seed=12)
    ctx = _ctx()
    bad = inst.extra["vtype"].copy()
    bad[5] = 3
    with pytest.raises(NysError):
        _solve(ctx, type(inst)(**{**inst.__dict__, "extra": {"vtype": bad, "ub": inst.extra["ub"]}}))
    ub = inst.extra["ub"].copy()
    ub[np.where(inst.extra["vtype"] == 2)[0][0]] = 0.0
    with pytest.raises(NysError):
        _solve(ctx, type(inst)(**{**inst.__dict__, "extra": {"vtype": inst.extra["vtype"], "ub": ub}}))
    ctx.close()


def test_general_multirank_loopback():
    """f1 on 2 loopback ranks (column shards of A with their vtype / ub shards)."""
    import concurrent.futures as cf
    from paper_2404_14524_b200 import Context, LoopbackComm, colmajor_device
    inst = make_general(150, 700, 0.2, 0.3, ell=20, seed=13)
    vt, u = inst.extra["vtype"], inst.extra["ub"]
    world, m, n = 2, inst.m, inst.n
    comm = LoopbackComm(world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    ctxs = [Context(0, stream=streams[r], nccl_id=comm.id, rank=r, world=world) for r in range(world)]
    bounds = [((n * r) // world, (n * (r + 1)) // world) for r in range(world)]
    data = []
    for lo, hi in bounds:
        Ad, lda = colmajor_device(np.asfortranarray(inst.A[:, lo:hi]))
        data.append((Ad, lda, dev(inst.q[lo:hi]), dev(inst.b), dev(inst.c[lo:hi]), dev(vt[lo:hi], torch.int8),
                     dev(u[lo:hi])))
    torch.cuda.synchronize()

    def worker(r):
        torch.cuda.set_device(0)
        Ad, lda, q, b, c, v, uu = data[r]
        with torch.cuda.stream(streams[r]):
            g = ctxs[r].nys_ipppmm_solve(Ad, lda, m, q, b, c, ell=inst.ell, vtype=v, ub=uu)
        streams[r].synchronize()
        return {k: _h(val) if hasattr(val, "cpu") else val for k, val in g.items() if k != "log"}

    try:
        with cf.ThreadPoolExecutor(max_workers=world) as ex:
            res = list(ex.map(worker, range(world)))
    finally:
        for cx in ctxs:
            cx.close()
        comm.close()
    ref = ippmm_gen.solve_general(inst.A, inst.q, inst.b, inst.c, vt, u, ippmm.Options(path="krylov", ell=inst.ell))
    for g in res:
        assert g["status"] == 0 and g["rel_p"] <= 1e-8 and g["rel_d"] <= 1e-8 and g["mu"] <= 1e-8
    assert np.array_equal(res[0]["y"], res[1]["y"]) and res[0]["inner"] == res[1]["inner"]
    x = np.concatenate([g["x"] for g in res])
    z = np.concatenate([g["z"] for g in res])
    s = np.concatenate([g["s"] for g in res])
    band_ = (band_general(inst, x, res[0]["y"], z, s, res[0]["obj"], res[0]["dual_obj"]) +
              band_general(inst, ref.x, ref.y, ref.z, ref.s, ref.obj, ref.dual_obj))
    tol = 1e-7 * max(1.0, abs(ref.obj))   # strict (north_star); the certified band is only reported
    print(f"obj diff vs oracle: strict tol {tol:.3e}, certified bands {band_:.3e}")
    assert abs(res[0]["obj"] - ref.obj) <= tol
    assert abs(res[0]["outer"] - ref.outer) <= 2


def test_general_all_free_is_the_kkt_solution():
    """Reading G5 on the GPU: every variable free -> the equality-constrained QP's KKT solution."""
    rs = np.random.default_rng(9)
    m, n = 30, 70
    A = rs.standard_normal((m, n))
    q = rs.uniform(0.5, 2.0, n)
    b = rs.standard_normal(m)
    c = rs.standard_normal(n)
    K = np.block([[np.diag(q), A.T], [A, np.zeros((m, m))]])
    sol = np.linalg.solve(K, np.concatenate([-c, b]))
    x_kkt, y_kkt = sol[:n], -sol[n:]
    from paper_2404_14524_b200 import colmajor_device
    ctx = _ctx()
    Ad, lda = colmajor_device(A)
    g = ctx.nys_ipppmm_solve(Ad, lda, m, dev(q), dev(b), dev(c), ell=8,
                             vtype=torch.ones(n, dtype=torch.int8, device="cuda"), ub=dev(np.zeros(n)))
    torch.cuda.synchronize()
    assert g["status"] == 0
    assert np.abs(_h(g["x"]) - x_kkt).max() <= 1e-7 and np.abs(_h(g["y"]) - y_kkt).max() <= 1e-7
    assert np.all(_h(g["z"]) == 0)
    ctx.close()


@pytest.mark.parametrize("kw", [dict(prec_refresh=3), dict(ell_max=64), dict(precond=1)])
def test_general_form_with_reuse_adaptive_and_chol(kw):
    """f1 combined with f3 (reuse, adaptive rank) and f2 (partial Cholesky): the same optimum (KKT of
    (P~)/(D~) at 1e-8 and the objective within the certified bands of the plain solve)."""
    inst = make_general(150, 600, 0.2, 0.3, ell=16, seed=14)
    vt, u = inst.extra["vtype"], inst.extra["ub"]
    J = vt == 2
    ctx = _ctx()
    g0 = _solve(ctx, inst)
    g = _solve(ctx, inst, **kw)
    torch.cuda.synchronize()
    assert g0["status"] == 0 and g["status"] == 0
    x, y, z, w, s = (_h(g[k]) for k in ("x", "y", "z", "w", "s"))
    bn = np.sqrt(inst.b @ inst.b + u[J] @ u[J])
    rP = np.concatenate([inst.b - inst.A @ x, (u - x - w)[J]])
    assert np.linalg.norm(rP) / (1 + bn) <= 1.01e-8
    assert np.linalg.norm(inst.c + inst.q * x - inst.A.T @ y - z + s) / (1 + np.linalg.norm(inst.c)) <= 1.01e-8
    assert abs(g["obj"] - g0["obj"]) <= 1e-7 * max(1.0, abs(g0["obj"]))
    ctx.close()
