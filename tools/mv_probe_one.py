"""One fused normal matvec at m x n against a float64 host reference (debug probe; prints the plan with NYS_DEBUG=1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context, colmajor_device  # noqa: E402

m, n = (int(x) for x in sys.argv[1].split("x"))
ctx = Context(0)
rs = np.random.default_rng(0)
A = rs.standard_normal((m, n))
Ad, lda = colmajor_device(A)
d, v = rs.uniform(0.1, 2, n), rs.standard_normal(m)
w = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
ctx.nys_normal_matvec(Ad, lda, m, torch.from_numpy(d).cuda(), None, 0.3, torch.from_numpy(v).cuda(), w)
torch.cuda.synchronize()
ref = A @ (d * (A.T @ v)) + 0.3 * v
print(f"m={m} n={n}: rel err {np.linalg.norm(w.cpu().numpy() - ref) / np.linalg.norm(ref):.3e}", flush=True)
