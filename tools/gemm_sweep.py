"""Sketch GEMM tuning sweep: kernel family (64x64 cp.async / 128-row TMA / 128-row cp.async) x split-K of
each of the two products (T = A^T Omega: NYS_GEMM_SPLITS_K, Y = A T: NYS_GEMM_SPLITS_M; 0 = the
library's heuristic), nys_sketch_apply timed with CUDA events (median of 9), against cuBLAS.
Usage: gemm_sweep.py MxNxELL [MxNxELL ...]"""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context  # noqa: E402

st = torch.cuda.Stream()
ctx = Context(0, stream=st)
FAM = {"old64": {"NYS_GEMM_OLD": "1"}, "nt_tma": {"NYS_GEMM_NT_MIN": "0,0"},
       "nt_cp": {"NYS_GEMM_NT_MIN": "0,0", "NYS_GEMM_CPASYNC": "1"}, "default": {}}
KEYS = ["NYS_GEMM_OLD", "NYS_GEMM_NT_MIN", "NYS_GEMM_CPASYNC", "NYS_GEMM_SPLITS_K", "NYS_GEMM_SPLITS_M"]


def timed(fn, R=9):
    with torch.cuda.stream(st):
        fn()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            fn()
            b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
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
        T = torch.empty((n, ell), dtype=torch.float64, device="cuda")
        Yt = torch.empty((ell, m), dtype=torch.float64, device="cuda")

    def cublas():
        torch.matmul(A[:, :m], Om[:, :m].t(), out=T)
        T.mul_(d[:, None])
        torch.matmul(T.t(), A[:, :m], out=Yt)

    t_cb = timed(cublas)
    res = []
    for fam, env in FAM.items():
        for sk, sm in itertools.product([0, 1, 2, 4, 8, 16], [0, 2, 4, 8, 16, 32]):
            if fam == "default" and (sk or sm):
                continue
            for k in KEYS:
                os.environ.pop(k, None)
            os.environ.update(env)
            if sk:
                os.environ["NYS_GEMM_SPLITS_K"] = str(sk)
            if sm:
                os.environ["NYS_GEMM_SPLITS_M"] = str(sm)
            t = timed(lambda: ctx.nys_sketch_apply(A, lda, m, d, None, ell, Om, Y))
            res.append((t, fam, sk, sm))
    for k in KEYS:
        os.environ.pop(k, None)
    res.sort()
    dflt = [r for r in res if r[1] == "default"][0][0]
    print(f"m={m} n={n} ell={ell}: cuBLAS {t_cb * 1e3:.1f} us, library default {dflt * 1e3:.1f} us; best:", flush=True)
    for t, fam, sk, sm in res[:8]:
        print(f"   {t * 1e3:8.1f} us  {fam:7s} splits_K={sk} splits_M={sm}  ({t_cb / t:.2f}x cuBLAS)", flush=True)
    del A, Om, Y, T, Yt
    torch.cuda.empty_cache()
