"""Sketch GEMMs (nys_sketch_apply: T = d o (A^T Omega), Y = A T; 4 m n l flops) against the same two
products through cuBLAS (torch.matmul fp64 = DGEMM) on the same device-resident operands, CUDA events,
median of R.  Usage: gemm_vs_cublas.py MxNxELL [MxNxELL ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context  # noqa: E402

R = 7
st = torch.cuda.Stream()
ctx = Context(0, stream=st)


def timed(fn):
    with torch.cuda.stream(st):
        fn()
        fn()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            fn()
            b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


for shape in sys.argv[1:]:
    m, n, ell = (int(x) for x in shape.split("x"))
    lda = (m + 31) // 32 * 32
    mp = m + (m % 2)
    with torch.cuda.stream(st):
        A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
        d = torch.rand(n, dtype=torch.float64, device="cuda") + 0.1
        Om = torch.empty((ell, mp), dtype=torch.float64, device="cuda")
        ctx.nys_gaussian(m, ell, 0, 1, Om)
        Y = torch.empty((ell, mp), dtype=torch.float64, device="cuda")
        At = A[:, :m]                      # n x m = A^T (row-major view of the column-major A)
        Omt = Om[:, :m]                    # ell x m = Omega^T
        T = torch.empty((n, ell), dtype=torch.float64, device="cuda")
        Yt = torch.empty((ell, m), dtype=torch.float64, device="cuda")

    def lib():
        ctx.nys_sketch_apply(A, lda, m, d, None, ell, Om, Y)

    def cublas():
        torch.matmul(At, Omt.t(), out=T)
        T.mul_(d[:, None])
        torch.matmul(T.t(), At, out=Yt)

    fl = 4.0 * m * n * ell
    t_lib = timed(lib)
    t_cb = timed(cublas)
    with torch.cuda.stream(st):
        err = float((Y[:, :m] - Yt).norm() / Yt.norm())
    st.synchronize()
    print(f"m={m} n={n} ell={ell}: library {t_lib * 1e3:.3f} ms = {fl / t_lib / 1e12:.2f} TFLOP/s; "
          f"cuBLAS (2 DGEMM + scale) {t_cb * 1e3:.3f} ms = {fl / t_cb / 1e12:.2f} TFLOP/s; "
          f"library/cuBLAS speed {t_cb / t_lib:.2f}x; rel diff {err:.1e}", flush=True)
    del A, Om, Y, T, Yt
    torch.cuda.empty_cache()
