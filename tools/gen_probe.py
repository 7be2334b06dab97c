import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle import ippmm, ippmm_gen
from synth import make_general, make_config
from paper_2404_14524_b200 import Context, colmajor_device
dev = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(dt).cuda()
ctx = Context(0)
def show(g, ref):
    for k in range(min(len(g["log"]), len(ref.log))):
        a, b = g["log"][k], ref.log[k]
        print(f"k={k} mu {a['mu']:.10e} {b['mu']:.10e} ap {a['alpha_p']:.8f} {b['alpha_p']:.8f} ad {a['alpha_d']:.8f} {b['alpha_d']:.8f} pcg {a['pcg_pred']}/{a['pcg_corr']} {b['pcg_pred']}/{b['pcg_corr']}")
inst = make_config(1, m=200, n=800, ell=20)
Ad, lda = colmajor_device(inst.A)
g = ctx.nys_ipppmm_solve(Ad, lda, inst.m, dev(inst.q), dev(inst.b), dev(inst.c), ell=inst.ell)
ref = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell))
print("== standard cfg1"); show(g, ref)
g = ctx.nys_ipppmm_solve(Ad, lda, inst.m, dev(inst.q), dev(inst.b), dev(inst.c), ell=inst.ell, vtype=torch.zeros(inst.n, dtype=torch.int8, device='cuda'))
print("== gen all-I cfg1"); show(g, ref)
for (m, n, ff, fb, ell) in [(100, 300, 0.2, 0.3, 20), (50, 400, 0.0, 1.0, 20), (80, 240, 1/3, 0.0, 20)]:
    inst = make_general(m, n, ff, fb, ell=ell)
    vt, u = inst.extra["vtype"], inst.extra["ub"]
    Ad, lda = colmajor_device(inst.A)
    g = ctx.nys_ipppmm_solve(Ad, lda, inst.m, dev(inst.q), dev(inst.b), dev(inst.c), ell=ell, vtype=dev(vt, torch.int8), ub=dev(u))
    ref = ippmm_gen.solve_general(inst.A, inst.q, inst.b, inst.c, vt, u, ippmm.Options(path="krylov", ell=ell))
    print("== gen", m, n, ff, fb); show(g, ref)
