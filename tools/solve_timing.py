"""Per-solve device time (CUDA events around each nys_ipppmm_solve call) against the library's own
host wall clock t_total_ms, to locate time spent outside the C solve.  Usage: solve_timing.py CFG [K]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context, colmajor_device  # noqa: E402
from synth import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
inst = make_config(cfg)
st = torch.cuda.Stream()
ctx = Context(0, stream=st)
Ad, lda = colmajor_device(inst.A)
dv = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
q, b, c = dv(inst.q), dv(inst.b), dv(inst.c)


def solve():
    with torch.cuda.stream(st):
        return ctx.nys_ipppmm_solve(Ad, lda, inst.m, q, b, c, ell=inst.ell)


for _ in range(3):
    solve()
torch.cuda.synchronize()
keep = []
for i in range(K):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(st)
    g = solve()
    e1.record(st)
    h1 = time.perf_counter()
    e1.synchronize()
    keep.append(g)
    print(f"cfg{cfg} solve {i}: events {e0.elapsed_time(e1):.2f} ms, host call {1e3 * (h1 - h0):.2f} ms, "
          f"t_total {g['t_total_ms']:.2f} ms (sketch {g['t_sketch_ms']:.2f}, pcg {g['t_pcg_ms']:.2f}, "
          f"other {g['t_other_ms']:.2f}), outer {g['outer']}, inner {g['inner']}", flush=True)
