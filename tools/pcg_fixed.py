import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import make_config
from paper_2404_14524_b200 import Context, colmajor_device
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
inst = make_config(cfg)
st = torch.cuda.Stream()
ctx = Context(0, stream=st)
Ad, lda = colmajor_device(inst.A)
m, ell = inst.m, inst.ell
mp = m + (m % 2)
rs = np.random.default_rng(0)
dv = lambda a: torch.from_numpy(a).cuda()
d = dv(rs.uniform(0.01, 2.0, inst.n)); rhs = dv(rs.standard_normal(m)); x = torch.zeros(m, dtype=torch.float64, device="cuda")
Om = torch.empty((ell, mp), dtype=torch.float64, device="cuda"); U = torch.empty_like(Om); lam = torch.empty(ell, dtype=torch.float64, device="cuda")
with torch.cuda.stream(st):
    ctx.nys_gaussian(m, ell, 0, 1, Om)
    ctx.nys_sketch(Ad, lda, m, d, None, 1e-2, ell, Om, U, lam)
    for _ in range(3):
        info = ctx.nys_pcg_solve(Ad, lda, m, d, None, 1e-2, ell, U, lam, 1e-2, rhs, x, 0.0, iters)
torch.cuda.synchronize()
print("iters", info.iters, "ms", info.t_ms)
