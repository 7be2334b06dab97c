"""Sketch timing on a device-generated A (m x n, fp64): nys_sketch_apply (the two DMMA GEMMs, 4 m n l flops)
and nys_sketch (plus the Nystrom factorisation), CUDA events, median of R.  Usage: sketch_bench.py MxN ELL [R]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context  # noqa: E402

m, n = (int(x) for x in sys.argv[1].split("x"))
ell = int(sys.argv[2])
R = int(sys.argv[3]) if len(sys.argv) > 3 else 5
st = torch.cuda.Stream()
ctx = Context(0, stream=st)
lda = (m + 31) // 32 * 32
mp = m + (m % 2)
with torch.cuda.stream(st):
    A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
    d = torch.rand(n, dtype=torch.float64, device="cuda") + 0.1
    Om = torch.empty((ell, mp), dtype=torch.float64, device="cuda")
    ctx.nys_gaussian(m, ell, 0, 1, Om)
    Y = torch.empty((ell, mp), dtype=torch.float64, device="cuda")
    U = torch.empty((ell, mp), dtype=torch.float64, device="cuda")
    lam = torch.empty(ell, dtype=torch.float64, device="cuda")


def timed(fn):
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            fn()
            b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts)), float(min(ts))


with torch.cuda.stream(st):
    ctx.nys_sketch_apply(A, lda, m, d, None, ell, Om, Y)
t_apply, t_apply_min = timed(lambda: ctx.nys_sketch_apply(A, lda, m, d, None, ell, Om, Y))
with torch.cuda.stream(st):
    info = ctx.nys_sketch(A, lda, m, d, None, 1e-3, ell, Om, U, lam)
print(f"jacobi sweeps {info.jacobi_sweeps}, chol retries {info.chol_retries}, orth err {info.orth_err:.2e}")
t_sk, t_sk_min = timed(lambda: ctx.nys_sketch(A, lda, m, d, None, 1e-3, ell, Om, U, lam))
fl = 4.0 * m * n * ell
print(f"m={m} n={n} ell={ell}: sketch GEMMs {t_apply * 1e3:.2f} ms (min {t_apply_min * 1e3:.2f}) = {fl / t_apply / 1e12:.2f} "
      f"TFLOP/s (best {fl / t_apply_min / 1e12:.2f}); sketch + factorisation {t_sk * 1e3:.2f} ms -> factorisation "
      f"{(t_sk - t_apply) * 1e3:.2f} ms", flush=True)
