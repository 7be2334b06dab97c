"""Probe: which output rows of the normal matvec stay unwritten (NaN-poisoned output) for large m."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2404_14524_b200 import Context, colmajor_device
ctx = Context(0)
rs = np.random.default_rng(0)
for m, n in [(70000, 33), (70000, 17), (70000, 200), (50000, 33), (50000, 301), (20000, 40), (139264, 9), (100000, 64), (60000, 33)]:
    A = rs.standard_normal((m, n))
    Ad, lda = colmajor_device(A)
    d, v = rs.uniform(0.1, 2, n), rs.standard_normal(m)
    ref = A @ (d * (A.T @ v)) + 0.3 * v
    res = []
    for rep in range(4):
        w = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
        ctx.nys_normal_matvec(Ad, lda, m, torch.from_numpy(d).cuda(), None, 0.3, torch.from_numpy(v).cuda(), w)
        torch.cuda.synchronize()
        wh = w.cpu().numpy()
        bad = np.nonzero(~np.isfinite(wh) | (np.abs(wh - ref) > 1e-9 * np.abs(ref).max()))[0]
        res.append(f"{len(bad)}" + (f"[{bad.min()}..{bad.max()}]" if len(bad) else ""))
    print(f"m={m} n={n}: bad rows per rep {res}", flush=True)
