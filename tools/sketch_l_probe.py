import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import make_svm_dual
from paper_2404_14524_b200 import Context, colmajor_device
ctx = Context(0)
inst = make_svm_dual(801, 20531)
B = inst.extra["B"]; m = B.shape[0]
Bd, lda = colmajor_device(B)
rs = np.random.default_rng(0)
d = torch.from_numpy(np.exp(rs.uniform(0, np.log(1e6), B.shape[1]))).cuda()
e = torch.full((m,), 0.3, dtype=torch.float64, device="cuda")
ells = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "50,100,128,160,200,256").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for ell in ells:
    Om = torch.empty((ell, m + (m % 2)), dtype=torch.float64, device="cuda")
    ctx.nys_gaussian(m, ell, 0, 1, Om)
    U = torch.empty_like(Om); lam = torch.empty(ell, dtype=torch.float64, device="cuda")
    info = ctx.nys_sketch(Bd, lda, m, d, e, 1e-3, ell, Om, U, lam)
    torch.cuda.synchronize()
    t = time.time()
    for _ in range(reps):
        info = ctx.nys_sketch(Bd, lda, m, d, e, 1e-3, ell, Om, U, lam)
    torch.cuda.synchronize()
    print(ell, "sweeps", info.jacobi_sweeps, "orth", info.orth_err, "retries", info.chol_retries, "ms/sketch", (time.time()-t)/reps*1e3, flush=True)
