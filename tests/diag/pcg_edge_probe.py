"""Cluster vs graph PCG against the oracle on edge shapes, error vs iteration count."""
import os, sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2404_14524_b200 import Context, colmajor_device
from oracle import linops, nystrom, rng as orng
from oracle.pcg import pcg as oracle_pcg
ctx = Context(0)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
def dev_cm(U):
    return dev(np.asarray(U, dtype=np.float64).T.copy())
for (m, n, ell, use_e) in [(30001, 10, 16, True), (30001, 40, 16, True), (20000, 300, 256, False), (138240, 24, 8, True)]:
    rs = np.random.default_rng(m + n + ell)
    A = rs.standard_normal((m, n)) / np.sqrt(n)
    d = rs.uniform(0.01, 2.0, n)
    e = rs.uniform(0.0, 1.0, m) if use_e else None
    delta = 1e-3
    rhs = rs.standard_normal(m)
    Om = orng.gaussian_omega(m, ell, 0, 1)
    Uo, lamo, _ = nystrom.nystrom_from_sketch(linops.sketch(A, d, Om, e), Om)
    pinv = lambda v: nystrom.precond_inv_apply(Uo, lamo, delta, v)
    Ad, lda = colmajor_device(A)
    for iters in (2, 4, 8, 15):
        xo, io = oracle_pcg(lambda v: linops.normal_matvec(A, d, v, delta, e), rhs, pinv, tol_abs=0.0, max_iter=iters)
        res = np.linalg.norm(linops.normal_matvec(A, d, xo, delta, e) - rhs)
        out = []
        for path in ("cluster", "graph"):
            if path == "graph": os.environ["NYS_NO_PCG_CLUSTER"] = "1"
            else: os.environ.pop("NYS_NO_PCG_CLUSTER", None)
            xg = torch.empty(m, dtype=torch.float64, device="cuda")
            ctx.nys_pcg_solve(Ad, lda, m, dev(d), dev(e) if use_e else None, delta, ell, dev_cm(Uo), dev(lamo), delta, dev(rhs), xg, 0.0, iters)
            xg = xg.cpu().numpy()
            out.append(np.linalg.norm(xg - xo) / np.linalg.norm(xo))
        print(f"m={m} n={n} ell={ell} it={iters}: oracle res {res:.2e}; cluster err {out[0]:.2e} graph err {out[1]:.2e}", flush=True)
