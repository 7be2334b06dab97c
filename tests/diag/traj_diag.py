"""Diagnostic: GPU vs oracle per-outer-iteration logs side by side for one IP-PMM case (prints only)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_14524_b200 import Context, colmajor_device
from oracle import ippmm
from synth import make_config

cfg, m, n, ell = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
kw = dict(a.split("=") for a in sys.argv[5:])
okw = {k: (float(v) if "." in v else int(v)) for k, v in kw.items()}
inst = make_config(cfg, m=m, n=n, ell=ell)
ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=ell, **okw))
ctx = Context(0)
Ad, lda = colmajor_device(inst.A)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
g = ctx.nys_ipppmm_solve(Ad, lda, inst.m, dv(inst.q), dv(inst.b), dv(inst.c), ell=ell, **okw)
print(f"{inst.name} {okw}: gpu obj {g['obj']!r} outer {g['outer']} inner {g['inner']} | ref {ref.obj!r} outer {ref.outer} inner {ref.inner_total}")
for k in range(max(len(g["log"]), len(ref.log))):
    a = g["log"][k] if k < len(g["log"]) else None
    b = ref.log[k] if k < len(ref.log) else None
    fa = f"mu {a['mu']:.10e} ap {a['alpha_p']:.12f} ad {a['alpha_d']:.12f} pcg {a['pcg_pred']:4d},{a['pcg_corr']:4d} built {a['prec_built']}" if a else "-"
    fb = f"mu {b['mu']:.10e} ap {b['alpha_p']:.12f} ad {b['alpha_d']:.12f} pcg {b['pcg_pred']:4d},{b['pcg_corr']:4d} built {int(b['prec_built'])}" if b else "-"
    flag = "" if (a and b and (a['pcg_pred'], a['pcg_corr']) == (b['pcg_pred'], b['pcg_corr']) and abs(a['mu'] - b['mu']) <= 1e-9 * b['mu']) else "  <<<"
    print(f"k={k:3d} GPU {fa} | REF {fb}{flag}")
