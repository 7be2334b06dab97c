"""Fused normal matvec (nys_normal_matvec, incl. its finalize) time vs shape on device-generated A,
CUDA events, median of 5 runs of 20 back-to-back calls.  Usage: mv_sweep.py MxN [MxN ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context  # noqa: E402

st = torch.cuda.Stream()
ctx = Context(0, stream=st)
for shape in sys.argv[1:]:
    m, n = (int(x) for x in shape.split("x"))
    lda = (m + 31) // 32 * 32
    with torch.cuda.stream(st):
        A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
        d = torch.rand(n, dtype=torch.float64, device="cuda") + 0.1
        e = torch.rand(m, dtype=torch.float64, device="cuda") + 0.5
        v = torch.randn(m, dtype=torch.float64, device="cuda")
        w = torch.empty(m, dtype=torch.float64, device="cuda")
        for _ in range(3):
            ctx.nys_normal_matvec(A, lda, m, d, e, 1e-3, v, w)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            for _ in range(20):
                ctx.nys_normal_matvec(A, lda, m, d, e, 1e-3, v, w)
            b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 20)
    t = float(np.median(ts))
    by = 8.0 * (m * n + n + 3 * m)
    print(f"m={m} n={n} CL={os.environ.get('NYS_MV_CL', '-')}: {t:.1f} us, {by / t / 1e3:.0f} GB/s", flush=True)
    del A
    torch.cuda.empty_cache()
