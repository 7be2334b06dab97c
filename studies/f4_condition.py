"""§8(f) f4 / paper §5.2.2: condition numbers of N_delta = N_k + delta_k I before and
after preconditioning at the IP-PMM iterations where the relative primal / dual infeasibilities and
mu first fall below eps in {1e-2, 1e-4, 1e-6, 1e-8}, for the Nystrom preconditioner (Alg. 1-2) and
the partial Cholesky preconditioner of ranks ell.

Workload: the paper's dual-SVM formulation (App. C.2) on a synthetic CIFAR10-shaped 1000-sample
subset (d = 3072 features -> normal equations 3073 x 3073), synth.make_svm_dual.
The iterates come from the library's own solve (nys_ipppmm_solve, re-run with max_outer = k to
read the iterate of iteration k); U, Lambda from nys_sketch; the partial Cholesky P^{-1} from
nys_partial_cholesky + nys_chol_precond_apply on the unit vectors.  Dense eigensolves use
torch.linalg.eigvalsh (cuSOLVER) in fp64.

    python -m studies.f4_condition [--samples 1000] [--d 3072] [--ells 10,20,50,100,200,256]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=1000)
    ap.add_argument("--d", type=int, default=3072)
    ap.add_argument("--ells", default="10,20,50,100,200,256")
    ap.add_argument("--solve-ell", type=int, default=50)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2404_14524_b200 import Context, colmajor_device
    from synth import make_svm_dual
    ells = [int(v) for v in args.ells.split(",")]
    inst = make_svm_dual(args.samples, args.d, ell=args.solve_ell)
    dev = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(dt).cuda()  # noqa: E731
    B = inst.extra["B"]
    m, nb = B.shape
    vt, ub = inst.extra["vtype"], inst.extra["ub"]
    Bd, lda = colmajor_device(B)
    ctx = Context(0)
    kw = dict(structure=2, unit_blocks=inst.extra["unit_blocks"], vtype=dev(vt, torch.int8), ub=dev(ub))
    qd, bd, cd = dev(inst.q), dev(inst.b), dev(inst.c)
    full = ctx.nys_ipppmm_solve(Bd, lda, m, qd, bd, cd, ell=args.solve_ell, **kw)
    log = full["log"]
    print(f"solve: status {full['status']} outer {full['outer']} inner {full['inner']}", flush=True)
    B_t = torch.from_numpy(B).cuda()
    rows = []
    for eps in (1e-2, 1e-4, 1e-6, 1e-8):
        k = next((r["k"] for r in log if max(r["rel_p"], r["rel_d"], r["mu"]) <= eps), None)
        if k is None:
            k = full["outer"]                                        # reached at the final check
            rec = None
        else:
            rec = log[k]
        it = ctx.nys_ipppmm_solve(Bd, lda, m, qd, bd, cd, ell=args.solve_ell, max_outer=k, **kw)
        x, z, w, s = (it[v].double() for v in ("x", "z", "w", "s"))
        rho = rec["rho"] if rec else log[-1]["rho"]
        delta = rec["delta"] if rec else log[-1]["delta"]
        vtt = dev(vt, torch.int8)
        th = torch.where(vtt == 1, torch.zeros_like(x), z / x)
        th = th + torch.where(vtt == 2, s / w, torch.zeros_like(x))
        dfull = 1.0 / (qd + th + rho)                                  # D = (Q + Theta^{-1} + rho I)^{-1}
        dB, dU = dfull[:nb].contiguous(), dfull[nb:]
        e = torch.zeros(m, dtype=torch.float64, device="cuda")
        e[:args.d] = dU                                               # the identity block's diagonal term
        N = (B_t * dB[None, :]) @ B_t.T + torch.diag(e)
        Nd = N + delta * torch.eye(m, dtype=torch.float64, device="cuda")
        ev = torch.linalg.eigvalsh(Nd)
        kap = float(ev[-1] / ev[0])
        row = {"eps": eps, "k": k, "rho": rho, "delta": delta, "kappa_N": kap, "nystrom": {}, "chol": {}}
        for ell in ells:
            Om = torch.empty((ell, m), dtype=torch.float64, device="cuda")
            U = torch.empty((ell, m), dtype=torch.float64, device="cuda")
            lam = torch.empty(ell, dtype=torch.float64, device="cuda")
            ctx.nys_gaussian(m, ell, 11, k + 1, Om)
            ctx.nys_sketch(Bd, lda, m, dB, e, delta, ell, Om, U, lam)
            torch.cuda.synchronize()
            Ut = U.T                                                  # m x ell
            mu = delta                                                # mu_prec = delta_k (A7)
            # P^{-1/2} = sqrt(lam_l + mu) U (Lam + mu)^{-1/2} U^T + I - U U^T  (eq. P:418)
            coef = torch.sqrt((lam[-1] + mu) / (lam + mu)) - 1.0
            Ph = torch.eye(m, dtype=torch.float64, device="cuda") + (Ut * coef[None, :]) @ Ut.T
            ev_n = torch.linalg.eigvalsh(Ph @ Nd @ Ph)
            row["nystrom"][ell] = float(ev_n[-1] / ev_n[0])
            # partial Cholesky: P^{-1} columns by applying it to the unit vectors
            ctx.nys_partial_cholesky(Bd, lda, m, dB, e, delta, ell)
            Pinv = torch.empty((m, m), dtype=torch.float64, device="cuda")
            I = torch.eye(m, dtype=torch.float64, device="cuda")
            for i in range(m):
                ctx.nys_chol_precond_apply(m, I[i], Pinv[i])
            torch.cuda.synchronize()
            Pinv = 0.5 * (Pinv + Pinv.T)
            C = torch.linalg.cholesky(Pinv)
            ev_c = torch.linalg.eigvalsh(C.T @ Nd @ C)
            row["chol"][ell] = float(ev_c[-1] / ev_c[0])
        rows.append(row)
        print(f"eps {eps:.0e} k {k:2d} kappa(N_delta) {kap:.3e} | Nystrom " +
              " ".join(f"l={l}:{row['nystrom'][l]:.2e}" for l in ells) + " | Chol " +
              " ".join(f"l={l}:{row['chol'][l]:.2e}" for l in ells), flush=True)
    out = {"study": "f4 condition numbers (P:1058-1086)", "workload": inst.name, "m": m, "n": inst.n,
           "solve_ell": args.solve_ell, "outer": full["outer"], "rows": rows,
           "when": time.strftime("%Y-%m-%d %H:%M:%S")}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
