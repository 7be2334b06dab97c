"""Diagnostic: config-2 recipe (structure 1) GPU vs oracle trajectories over the first K outer iterations."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_14524_b200 import Context, colmajor_device
from oracle import ippmm, svm
from synth import make_config

ctx = Context(0)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
K = 3
for N, d, ell in [(10000, 200, 20), (10000, 200, 50), (12000, 100, 20), (16000, 64, 30), (9000, 150, 40), (20000, 100, 50)]:
    inst = make_config(2, m=N, n=d, ell=ell)
    op = svm.SvmOperator(inst.extra["Xt"])
    ref = ippmm.solve(op, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=ell, max_outer=K))
    Xd, lda = colmajor_device(inst.extra["Xt"])
    g = ctx.nys_ipppmm_solve(Xd, lda, N, dv(inst.q), dv(inst.b), dv(inst.c), ell=ell, structure=1, max_outer=K)
    rows = []
    ok = True
    for a, b in zip(g["log"], ref.log):
        same = (a["pcg_pred"], a["pcg_corr"]) == (b["pcg_pred"], b["pcg_corr"]) and abs(a["mu"] - b["mu"]) <= 1e-9 * b["mu"]
        ok &= same
        rows.append(f"{a['pcg_pred']},{a['pcg_corr']}/{b['pcg_pred']},{b['pcg_corr']} mu {abs(a['mu'] - b['mu']) / b['mu']:.1e}")
    ex = max(np.max(np.abs(g[k].cpu().numpy() - getattr(ref, k))) / max(1, np.max(np.abs(getattr(ref, k)))) for k in "xyz")
    print(f"N={N} d={d} ell={ell}: {'SAME' if ok else 'DIFF'} | " + " | ".join(rows) + f" | iterate err {ex:.2e}", flush=True)
