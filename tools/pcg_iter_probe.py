"""Per-iteration PCG time on a device-generated dense A (m x n, fp64) with e = 1 (config 2's operator
shape: m = 50000 rows, n = 1000 folded feature columns, ell = 100), against the fused normal matvec
alone.  CUDA events, median of R solves of ITERS iterations (tol 0: every solve runs ITERS).
Usage: pcg_iter_probe.py MxNxELL [ITERS] [R]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context  # noqa: E402

m, n, ell = (int(x) for x in sys.argv[1].split("x"))
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
R = int(sys.argv[3]) if len(sys.argv) > 3 else 5
st = torch.cuda.Stream()
ctx = Context(0, stream=st)
lda = (m + 31) // 32 * 32
mp = m + (m % 2)
with torch.cuda.stream(st):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((n, lda), dtype=torch.float64, device="cuda", generator=g) / np.sqrt(n)
    d = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 + 0.01
    e = torch.rand(m, dtype=torch.float64, device="cuda", generator=g) + 0.5
    rhs = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    x = torch.zeros(m, dtype=torch.float64, device="cuda")
    w = torch.empty(m, dtype=torch.float64, device="cuda")
    Om = torch.empty((ell, mp), dtype=torch.float64, device="cuda")
    U = torch.empty_like(Om)
    lam = torch.empty(ell, dtype=torch.float64, device="cuda")
    ctx.nys_gaussian(m, ell, 0, 1, Om)
    ctx.nys_sketch(A, lda, m, d, e, 1e-3, ell, Om, U, lam)


def timed(fn, reps):
    with torch.cuda.stream(st):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            fn()
            b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


t_mv = timed(lambda: [ctx.nys_normal_matvec(A, lda, m, d, e, 1e-3, rhs, w) for _ in range(20)], R) / 20
info = {}


def solve():
    info["i"] = ctx.nys_pcg_solve(A, lda, m, d, e, 1e-3, ell, U, lam, 1e-3, rhs, x, 0.0, iters)


t_pcg = timed(solve, R)
its = info["i"].iters
print(f"m={m} n={n} ell={ell} NYS_U_KEEP={os.environ.get('NYS_U_KEEP', '-')}: matvec {t_mv:.1f} us "
      f"({8.0 * (m * n + n + 3 * m) / t_mv / 1e3:.0f} GB/s); PCG {its} its {t_pcg / 1e3:.2f} ms = "
      f"{t_pcg / its:.1f} us/it (matvec share {t_mv * its / t_pcg:.2f})", flush=True)
