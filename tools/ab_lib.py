"""A/B one library build against another at config-1 shapes: nys_sketch (ell 20 / 50 / 64) and the full
solve.  Usage: python tools/ab_lib.py path/to/libnysipm.so  (run once per build, same box)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import _lib
_lib.load_library(sys.argv[1])
import numpy as np, torch
from synth import make_config
from paper_2404_14524_b200 import Context, colmajor_device
ctx = Context(0)
inst = make_config(1)
Ad, lda = colmajor_device(inst.A); m = inst.m
dev = lambda a: torch.from_numpy(a).cuda()
rs = np.random.default_rng(0)
d = torch.from_numpy(np.exp(rs.uniform(0, np.log(1e8), inst.A.shape[1]))).cuda()
e = torch.zeros(m, dtype=torch.float64, device="cuda")
for ell in [int(v) for v in os.environ.get("AB_ELLS", "20,50,64").split(",")]:
    Om = torch.empty((ell, m), dtype=torch.float64, device="cuda")
    ctx.nys_gaussian(m, ell, 0, 1, Om)
    U = torch.empty_like(Om); lam = torch.empty(ell, dtype=torch.float64, device="cuda")
    info = ctx.nys_sketch(Ad, lda, m, d, e, 1e-6, ell, Om, U, lam)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record(); info = ctx.nys_sketch(Ad, lda, m, d, e, 1e-6, ell, Om, U, lam); s1.record(); s1.synchronize()
        ts.append(s0.elapsed_time(s1))
    Uh = U.cpu().numpy()
    print(f"ell {ell} sketch ms median {np.median(ts):.4f} min {min(ts):.4f} sweeps {info.jacobi_sweeps} orth {info.orth_err:.2e} "
          f"|UU^T-I| {np.linalg.norm(Uh @ Uh.T - np.eye(ell)):.2e} lam0 {lam[0].item():.12e} lam_l {lam[-1].item():.6e}", flush=True)
qs, bs, cs = dev(inst.q), dev(inst.b), dev(inst.c)
for r in range(4):
    t = time.time()
    sol = ctx.nys_ipppmm_solve(Ad, lda, m, qs, bs, cs, ell=inst.ell)
    torch.cuda.synchronize()
    print(f"solve {r}: {1e3*(time.time()-t):.2f} ms outer {sol['outer']} inner {sol['inner']} obj {sol['obj']!r} "
          f"sketch {sol['t_sketch_ms']:.2f} pcg {sol['t_pcg_ms']:.2f}", flush=True)
