"""Memory / race checks without compute-sanitizer (closed on the GPU pool: runs under it left GPUs
needing a reset).  Run with NYS_DEBUG_GUARD=1:

  * library workspaces: NaN-poisoned on allocation, followed by a 64 KiB canary checked after every
    ABI call (nys_ctx::check_guards) -> an out-of-bounds write past any workspace fails the call;
  * caller buffers: every output lives inside a larger allocation whose head and tail are filled with a
    sentinel, the output itself NaN-poisoned before the call -> checked here after the call: no write
    outside the output, every output element written (no NaN left), no NaN produced from poisoned
    workspace reads;
  * races: every case runs REPEATS times; the outputs must be bitwise identical (shared-memory / grid
    races, mbarrier or DSMEM ordering bugs show up as run-to-run differences), and each is checked
    against a float64 host reference.

Cases cover every kernel family: fused matvec (whole-column and cluster/DSMEM split), sketch GEMMs +
CholQR3 + one-sided Jacobi (single CTA, block-cluster), persistent PCG (cooperative grid barriers),
persistent cluster PCG (m > 8192), graph-path PCG (conditional WHILE graph), partial Cholesky, capped Nys-IP-PMM solves (dense,
structured) and the loopback multi-rank path.  Exit code != 0 on any failure."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2404_14524_b200 import Context, colmajor_device  # noqa: E402
from synth import make_config  # noqa: E402

REPEATS = 3
GUARD = 4096
SENT = 1.2345e300
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
ctx = Context(0)
only = sys.argv[1:] or None
failures = []


class Guarded:
    """An output buffer of `shape` inside a sentinel-filled allocation; the payload is NaN-poisoned."""

    def __init__(self, *shape):
        n = int(np.prod(shape))
        self.full = torch.full((n + 2 * GUARD,), SENT, dtype=torch.float64, device="cuda")
        self.t = self.full[GUARD:GUARD + n].view(*shape)
        self.t.fill_(float("nan"))

    def check(self, name, allow_nan=False):
        torch.cuda.synchronize()
        h = self.full.cpu().numpy()
        if not (np.all(h[:GUARD] == SENT) and np.all(h[-GUARD:] == SENT)):
            failures.append(f"{name}: write outside the output buffer")
        bad = np.nonzero(np.isnan(h[GUARD:-GUARD]))[0]
        if not allow_nan and len(bad):
            failures.append(f"{name}: output not fully written / NaN from poisoned workspace ({len(bad)} entries, "
                            f"first {bad[:4].tolist()}, last {bad[-1]})")
        return self.t.cpu().numpy().copy()


def case(name):
    def deco(fn):
        if only is not None and name not in only:
            return fn
        outs = []
        for rep in range(REPEATS):
            outs.append(fn(np.random.default_rng(0)))
            torch.cuda.synchronize()
        for k in outs[0]:
            for r in range(1, REPEATS):
                if not np.array_equal(outs[0][k], outs[r][k], equal_nan=True):
                    failures.append(f"{name}/{k}: run {r} differs from run 0 (max |diff| "
                                    f"{np.nanmax(np.abs(outs[0][k] - outs[r][k])):.3e})")
        print(f"[case] {name}: {REPEATS} runs, outputs {sorted(outs[0])}", flush=True)
        return fn
    return deco


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@case("matvec")
def _(rs):
    out = {}
    for m, n in [(300, 999), (20000, 40), (8193, 70), (70000, 33)]:
        A = rs.standard_normal((m, n))
        Ad, lda = colmajor_device(A)
        d, v, e = rs.uniform(0.1, 2, n), rs.standard_normal(m), rs.uniform(0, 1, m)
        w = Guarded(m)
        ctx.nys_normal_matvec(Ad, lda, m, dv(d), dv(e), 0.3, dv(v), w.t)
        wh = w.check(f"matvec {m}x{n}")
        ref = A @ (d * (A.T @ v)) + e * v + 0.3 * v
        if rel(wh, ref) > 1e-12:
            failures.append(f"matvec {m}x{n}: rel err {rel(wh, ref):.2e}")
        out[f"w{m}"] = wh
    return out


@case("sketch")
def _(rs):
    out = {}
    for m, n, ell in [(400, 900, 20), (1500, 600, 100), (3000, 500, 200)]:
        A = rs.standard_normal((m, n))
        Ad, lda = colmajor_device(A)
        Om = torch.empty((ell, m), dtype=torch.float64, device="cuda")
        ctx.nys_gaussian(m, ell, 0, 1, Om)
        U, lam = Guarded(ell, m), Guarded(ell)
        info = ctx.nys_sketch(Ad, lda, m, dv(np.ones(n)), None, 1e-2, ell, Om, U.t, lam.t)
        Uh, lh = U.check(f"sketch U {ell}"), lam.check(f"sketch lam {ell}")
        if info.orth_err > 1e-12:
            failures.append(f"sketch {ell}: orth err {info.orth_err:.2e}")
        N = A @ A.T
        if rel((Uh.T * lh) @ Uh, N) > 1e-8 and ell >= min(m, n):
            failures.append(f"sketch {ell}: Nystrom error")
        out[f"U{ell}"], out[f"lam{ell}"] = Uh, lh
    return out


def _prec(Ad, lda, m, n, ell, d, rs):
    Om = torch.empty((ell, m), dtype=torch.float64, device="cuda")
    ctx.nys_gaussian(m, ell, 0, 1, Om)
    U = torch.empty((ell, m), dtype=torch.float64, device="cuda")
    lam = torch.empty(ell, dtype=torch.float64, device="cuda")
    ctx.nys_sketch(Ad, lda, m, d, None, 1e-3, ell, Om, U, lam)
    return U, lam


@case("pcg_persistent")
def _(rs):
    inst = make_config(1, m=300, n=1200, ell=20)
    Ad, lda = colmajor_device(inst.A)
    m, ell = inst.m, inst.ell
    d = dv(rs.uniform(0.1, 2, inst.n))
    U, lam = _prec(Ad, lda, m, inst.n, ell, d, rs)
    x = Guarded(m)
    ctx.nys_pcg_solve(Ad, lda, m, d, None, 1e-3, ell, U, lam, 1e-3, dv(rs.standard_normal(m)), x.t, 0.0, 10)
    return {"x": x.check("pcg_persistent x")}


def _pcg_large(rs, name):
    m, n, ell = 20000, 60, 30
    A = rs.standard_normal((m, n)) / np.sqrt(n)
    Ad, lda = colmajor_device(A)
    d = dv(rs.uniform(0.1, 2, n))
    U, lam = _prec(Ad, lda, m, n, ell, d, rs)
    x = Guarded(m)
    ctx.nys_pcg_solve(Ad, lda, m, d, dv(rs.uniform(0, 1, m)), 1e-3, ell, U, lam, 1e-3, dv(rs.standard_normal(m)),
                      x.t, 0.0, 6)
    return {"x": x.check(f"{name} x")}


@case("pcg_cluster")      # m > 8192: the persistent cluster kernel (cluster DSMEM exchange, grid barriers)
def _(rs):
    return _pcg_large(rs, "pcg_cluster")


@case("pcg_graph")        # the same solve through the conditional-WHILE graph path
def _(rs):
    os.environ["NYS_NO_PCG_CLUSTER"] = "1"
    try:
        return _pcg_large(rs, "pcg_graph")
    finally:
        del os.environ["NYS_NO_PCG_CLUSTER"]


@case("chol")
def _(rs):
    inst = make_config(1, m=300, n=1200, ell=30)
    Ad, lda = colmajor_device(inst.A)
    piv = torch.empty(30, dtype=torch.int64, device="cuda")
    L, dS = Guarded(30, inst.m), Guarded(inst.m)
    ctx.nys_partial_cholesky(Ad, lda, inst.m, dv(rs.uniform(0.1, 2, inst.n)), None, 1e-2, 30, piv, L.t, dS.t)
    o = Guarded(inst.m)
    ctx.nys_chol_precond_apply(inst.m, dv(rs.standard_normal(inst.m)), o.t)
    return {"L": L.check("chol L"), "dS": dS.check("chol dS"), "Pv": o.check("chol apply"),
            "piv": piv.cpu().numpy().astype(np.float64)}


@case("ipm")
def _(rs):
    inst = make_config(0)
    Ad, lda = colmajor_device(inst.A)
    g = ctx.nys_ipppmm_solve(Ad, lda, inst.m, dv(inst.q), dv(inst.b), dv(inst.c), ell=inst.ell, max_outer=3)
    gi = make_config(2, m=600, n=30, ell=10)
    Xd, lda2 = colmajor_device(gi.extra["Xt"])
    g2 = ctx.nys_ipppmm_solve(Xd, lda2, gi.m, dv(gi.q), dv(gi.b), dv(gi.c), ell=10, structure=1, max_outer=2)
    return {"x": g["x"].cpu().numpy(), "y": g["y"].cpu().numpy(), "x2": g2["x"].cpu().numpy()}


@case("loopback")
def _(rs):
    from paper_2404_14524_b200 import LoopbackComm
    inst = make_config(0)
    comm = LoopbackComm(2)
    half = inst.n // 2
    streams = [torch.cuda.Stream() for _ in range(2)]
    ctxs = [Context(0, stream=streams[r], nccl_id=comm.id, rank=r, world=2) for r in range(2)]
    out = [None, None]

    def worker(r):
        torch.cuda.set_device(0)
        lo, hi = (0, half) if r == 0 else (half, inst.n)
        with torch.cuda.stream(streams[r]):
            Ad, lda = colmajor_device(np.asfortranarray(inst.A[:, lo:hi]))
            out[r] = ctxs[r].nys_ipppmm_solve(Ad, lda, inst.m, dv(inst.q[lo:hi]), dv(inst.b), dv(inst.c[lo:hi]),
                                              ell=inst.ell, max_outer=2)
        streams[r].synchronize()
    ts = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for c in ctxs:
        c.close()
    comm.close()
    if out[0]["log"][1]["mu"] != out[1]["log"][1]["mu"]:
        failures.append("loopback: replicated decisions differ across ranks")
    return {"y0": out[0]["y"].cpu().numpy(), "y1": out[1]["y"].cpu().numpy()}


ctx.close()
print(f"[sanitize_cases] NYS_DEBUG_GUARD={os.environ.get('NYS_DEBUG_GUARD', '0')} failures: {len(failures)}")
for f in failures:
    print("  FAIL", f)
sys.exit(1 if failures else 0)
