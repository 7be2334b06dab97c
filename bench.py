#!/usr/bin/env python
"""Benchmark: Nys-IP-PMM time-to-1e-8 on BASELINE.json configs[1] (m=2000, n=8000, l=50) on B200,
with the fused fp64 normal matvec (the dominant kernel) reported against the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1]

A "step" is one complete Nys-IP-PMM solve to tol 1e-8 (every SURVEY §8(a) row: D-update,
sketch + Nystrom factorisation, PCG with the fused matvec and preconditioner, Newton RHS /
recovery, predictor-corrector, residuals/TC/PEU, initial point) with the problem resident in
HBM.  `value` = seconds per solve (time-to-1e-8, lower is better); `e2e` = the same solve through
the C ABI with HOST buffers (H2D of A, q, b, c and D2H of x, y, z inside the timed region).
Multi-GPU (torchrun, N > 1): A's columns are sharded over ranks (strong scaling of the same
problem); timing is on the device, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 A·D·Aᵀv matvec GB/s (% HBM peak) and Nys-IP-PMM time-to-1e-8 at 1/2/4/8 GPU"
# dram__bytes_read.sum + dram__bytes_write.sum per fused-matvec launch from `ncu --set full`
# (profiles/, per config); None until captured for that config
TRAFFIC = {1: 134.6e6}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu: int = 0):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        import statistics
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def load_instance(cfg: int, rank: int, world: int):
    from synth import make_config
    inst = make_config(cfg)
    n = inst.n
    lo, hi = (n * rank) // world, (n * (rank + 1)) // world
    return inst, lo, hi


def run_reference(args):
    """--impl reference: the CPU oracle (numpy/scipy fp64) as it stands, on this host's cores."""
    import numpy as np
    from oracle import ippmm
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    inst, _, _ = load_instance(args.config, 0, 1)
    K = min(args.steps, 2)
    W = min(args.warmup, 1)
    times = []
    res = None
    for i in range(W + K):
        t0 = time.perf_counter()
        res = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell))
        dt = time.perf_counter() - t0
        if i >= W:
            times.append(dt)
    v = float(np.mean(times))
    cores = os.cpu_count()
    sample = (f"full oracle Nys-IP-PMM solve of {inst.name} per step ({res.outer} outer / {res.inner_total} PCG "
              f"iterations); {K} timed + {W} warm-up of the requested {args.steps}+{args.warmup}")
    line = {"metric": METRIC, "value": v, "unit": "s", "impl": "reference", "n_gpus": args.gpus, "steps": K,
            "warmup": W, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": inst.name, "m": inst.m, "n": inst.n, "ell": inst.ell, "tol": 1e-8},
            "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--matvec-reps", type=int, default=50)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2404_14524_b200 import Context, colmajor_device, nccl_unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    else:
        nid = None
    stream = torch.cuda.Stream(local)
    ctx = Context(local, stream=stream, nccl_id=nid, rank=rank, world=world)

    inst, lo, hi = load_instance(args.config, rank, world)
    A_loc = np.asfortranarray(inst.A[:, lo:hi])
    Ad, lda = colmajor_device(A_loc, device=f"cuda:{local}")
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{local}")  # noqa: E731
    q, b, c = dv(inst.q[lo:hi]), dv(inst.b), dv(inst.c[lo:hi])
    m, nloc = inst.m, hi - lo

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def one_solve():
        with torch.cuda.stream(stream):
            return ctx.nys_ipppmm_solve(Ad, lda, m, q, b, c, ell=inst.ell)

    # ---- warm-up ------------------------------------------------------------------------------
    for _ in range(max(args.warmup, 3)):
        g = one_solve()
    assert g["status"] == 0, f"solve status {g['status']}"
    # ---- timed region: K complete solves, CUDA events on the library's stream ------------------
    barrier()
    launches0 = ctx.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        results = [one_solve() for _ in range(args.steps)]
        ev1.record(stream)
        barrier()
    launches = ctx.kernel_launches - launches0
    t_dev = ev0.elapsed_time(ev1) / 1e3
    if world > 1:
        tt = torch.tensor([t_dev], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
    sec_per_solve = t_dev / args.steps
    matvecs_per_solve = results[-1]["matvecs"]

    # ---- dominant kernel: fused normal matvec, timed live with CUDA events on its stream ------
    # The launches are captured in CUDA graphs (no host overhead between launches):
    #   warm = R back-to-back matvecs;  cold = R x (256 MB L2-flushing read + matvec) minus R x flush
    rs = np.random.default_rng(0)
    d = dv(rs.uniform(0.01, 2.0, nloc))
    v = dv(rs.standard_normal(m))
    w = torch.empty(m, dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.ones(32 * 1024 * 1024, dtype=torch.float64, device=f"cuda:{local}")  # 256 MB
    R = args.matvec_reps
    with torch.cuda.stream(stream):
        for _ in range(5):
            ctx.nys_normal_matvec(Ad, lda, m, d, None, 1e-3, v, w)
            flush.sum()
    barrier()

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(R):
                fn()
        return g

    def mv():
        ctx.nys_normal_matvec(Ad, lda, m, d, None, 1e-3, v, w)

    fl_out = torch.empty((), dtype=torch.float64, device=f"cuda:{local}")

    def fl():
        torch.sum(flush, dim=0, out=fl_out)

    g_warm = capture(mv)
    g_cold = capture(lambda: (fl(), mv()))
    g_flush = capture(fl)
    barrier()

    def timed(g):
        g.replay()
        barrier()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        with torch.cuda.stream(stream):
            g.replay()
        b_.record(stream)
        barrier()
        return a.elapsed_time(b_) / 1e3

    mv_warm_s = timed(g_warm) / R
    mv_s = (timed(g_cold) - timed(g_flush)) / R
    del g_warm, g_cold, g_flush, flush
    mv_bytes = 8.0 * (m * nloc + nloc + 2 * m)  # A once + d + v in + w out
    mv_gbs = mv_bytes / mv_s / 1e9
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"

    # ---- e2e: the same solve through the C ABI with host buffers --------------------------------
    A_host = np.zeros((nloc, lda))
    A_host[:, :m] = A_loc.T
    qh, bh, ch = inst.q[lo:hi].copy(), inst.b.copy(), inst.c[lo:hi].copy()
    barrier()
    t0 = time.perf_counter()
    E_STEPS = max(1, min(args.steps, 3))
    for _ in range(E_STEPS):
        with torch.cuda.stream(stream):
            ge = ctx.nys_ipppmm_solve(A_host, lda, m, qh, bh, ch, ell=inst.ell, host=True)
    barrier()
    t_e2e = (time.perf_counter() - t0) / E_STEPS
    if world > 1:
        tt = torch.tensor([t_e2e], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    h2d = 8 * (m * nloc + 2 * nloc + m)
    d2h = 8 * (2 * nloc + m)

    # ---- CPU oracle baseline (rank 0, N = 1 only; bounded sample) --------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import ippmm
        t0 = time.perf_counter()
        r = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell))
        tc = time.perf_counter() - t0
        cpu = {"value": tc, "unit": "s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"one full oracle solve of {inst.name} ({r.outer} outer, {r.inner_total} PCG iters, "
                         f"obj {r.obj:.12g} vs GPU {results[-1]['obj']:.12g})"}

    if rank == 0:
        last = results[-1]
        line = {
            "metric": METRIC, "value": sec_per_solve, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": sec_per_solve * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": inst.name, "m": m, "n": inst.n, "ell": inst.ell, "tol": 1e-8,
                       "parallelism": f"column-shard x{world}",
                       "l2": "inputs larger than L2 (A = %.0f MB vs 126 MB L2), A streamed with L2 evict_first" % (8 * m * inst.n / 1e6)},
            "clocks": clk.summary(),
            "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": mv_gbs, "peak": hbm, "unit": "GB/s", "frac": mv_gbs / hbm,
                         "traffic": TRAFFIC.get(args.config), "kernel": "fused normal matvec (matvec_kernel + mv_finalize), L2 flushed (256 MB read) before each launch, graph-captured",
                         "peak_source": peak_src, "bytes_per_launch": mv_bytes, "launch_us": mv_s * 1e6,
                         "warm_l2_gbs": mv_bytes / mv_warm_s / 1e9,
                         "pcg_effective_gbs": last["inner"] * mv_bytes / (last["t_pcg_ms"] / 1e3) / 1e9,
                         "share_of_step": matvecs_per_solve * mv_s / sec_per_solve},
            "solve": {"outer": last["outer"], "inner": last["inner"], "obj": last["obj"], "rel_p": last["rel_p"],
                      "rel_d": last["rel_d"], "mu": last["mu"], "matvecs": matvecs_per_solve,
                      "t_sketch_ms": last["t_sketch_ms"], "t_pcg_ms": last["t_pcg_ms"],
                      "t_other_ms": last["t_other_ms"], "kernel_launches": last["kernel_launches"]},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
