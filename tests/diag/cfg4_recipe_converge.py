"""Diagnostic: does BASELINE config 4's recipe (A = W H + 1e-2 G, q with 30 % zeros, aspect n = 8 m as
in the full problem) converge to 1e-8 at reduced sizes?  GPU solve (and, for the smallest, the
oracle) — prints status, outer / inner counts, times, objectives."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_14524_b200 import Context, colmajor_device  # noqa: E402
from synth import make_config  # noqa: E402

ctx = Context(0)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
sizes = [(int(a), int(b), int(c)) for a, b, c in (s.split("x") for s in sys.argv[1:])] or [(1000, 8000, 100), (2000, 16000, 200), (5000, 40000, 200)]
for m, n, ell in sizes:
    t0 = time.time()
    inst = make_config(4, m=m, n=n, ell=ell)
    tg = time.time() - t0
    Ad, lda = colmajor_device(inst.A)
    torch.cuda.synchronize()
    t0 = time.time()
    g = ctx.nys_ipppmm_solve(Ad, lda, m, dv(inst.q), dv(inst.b), dv(inst.c), ell=ell)
    torch.cuda.synchronize()
    t1 = time.time() - t0
    pc = [(r["pcg_pred"], r["pcg_corr"]) for r in g["log"]]
    print(f"m={m} n={n} ell={ell}: gen {tg:.1f}s | GPU status {g['status']} outer {g['outer']} inner {g['inner']} "
          f"{t1:.2f}s obj {g['obj']!r} rel_p {g['rel_p']:.1e} rel_d {g['rel_d']:.1e} mu {g['mu']:.1e}", flush=True)
    print("   pcg per outer:", pc, flush=True)
    if m * n <= 2e7 and "--oracle" in os.environ.get("DIAG_FLAGS", "--oracle"):
        from oracle import ippmm
        t0 = time.time()
        r = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=ell))
        print(f"   oracle: {r.status} outer {r.outer} inner {r.inner_total} {time.time() - t0:.1f}s obj {r.obj!r} "
              f"rel diff {abs(r.obj - g['obj']) / max(1, abs(r.obj)):.2e}", flush=True)
