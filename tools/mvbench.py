"""Matvec micro-benchmark (tool, not product): GB/s of the fused normal matvec at several shapes, each timed
as a CUDA graph of R launches, 5 replays (min / median reported), with nvidia-smi power / clocks sampled."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context  # noqa: E402

SHAPES = [(2000, 8000), (64, 200000), (50000, 50000), (8192, 200000), (20000, 100000), (4096, 400000),
          (1000, 1000000), (128, 4000000)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]]

torch.cuda.set_device(0)
st = torch.cuda.Stream()
ctx = Context(0, stream=st)
flush = torch.ones(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
fl_out = torch.empty((), dtype=torch.float64, device="cuda")


def smi():
    import subprocess
    q = "clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap"
    return subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                          capture_output=True, text=True).stdout.strip()


def timed_graph(fn, R, reps=1):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(R):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / R)
    return sorted(ts)[len(ts) // 2] if reps > 1 else ts[0], min(ts)


# read-only stream ceiling: sum over 4 GB
big = torch.ones(512 * 1024 * 1024, dtype=torch.float64, device="cuda")
with torch.cuda.stream(st):
    t = timed_graph(lambda: torch.sum(big, dim=0, out=fl_out), 5)[0]
print(json.dumps({"read_only_sum_4GB_gbs": big.numel() * 8 / t / 1e9}), flush=True)
del big

for m, n in SHAPES:
    lda = (m + 31) // 32 * 32
    A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
    d = torch.rand(n, dtype=torch.float64, device="cuda") + 0.1
    v = torch.randn(m, dtype=torch.float64, device="cuda")
    w = torch.empty(m, dtype=torch.float64, device="cuda")
    byts = 8.0 * (m * n + n + 2 * m)
    with torch.cuda.stream(st):
        for _ in range(3):
            ctx.nys_normal_matvec(A, lda, m, d, None, 1e-3, v, w)
        torch.cuda.synchronize()
        R = max(6, min(200, int(2e9 / byts)))
        tw, tmin = timed_graph(lambda: ctx.nys_normal_matvec(A, lda, m, d, None, 1e-3, v, w), R, reps=5)
        out = {"m": m, "n": n, "MB": byts / 1e6, "warm_us": tw * 1e6, "warm_gbs": byts / tw / 1e9,
               "best_gbs": byts / tmin / 1e9, "smi_after": smi()}
        if byts < 1e9:
            tc = timed_graph(lambda: (torch.sum(flush, dim=0, out=fl_out), ctx.nys_normal_matvec(A, lda, m, d, None, 1e-3, v, w)), R)[0]
            tf = timed_graph(lambda: torch.sum(flush, dim=0, out=fl_out), R)[0]
            out["cold_us"] = (tc - tf) * 1e6
            out["cold_gbs"] = byts / (tc - tf) / 1e9
    print(json.dumps(out), flush=True)
    del A
    torch.cuda.empty_cache()
