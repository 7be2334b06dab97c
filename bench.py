#!/usr/bin/env python
"""Benchmark: Nys-IP-PMM time-to-1e-8 on B200, with the fused fp64 normal matvec (the dominant
kernel) reported against the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Default workload (the headline, SURVEY §8(d) "the HBM headline"): BASELINE.json configs[4]
(m=50000, l=200) with --n-per-gpu columns per rank (default 50000: at N=1 the one-GPU slice of
SURVEY A25, A = 20 GB; at N=8 the full n=400000 problem, 160 GB) -> "scaling": "weak".  The slice
does not reach 1e-8 in bench time (its square noise block leaves a tail no rank-200 Nystrom
preconditioner removes: PCG hits its 20000-iteration cap from outer iteration 18 on),
so a config-4 step is the first --max-outer (default 3) outer iterations of Nys-IP-PMM, labelled so
in config.step.  --config 0|1|2|3 selects another BASELINE config (a step is then a complete solve
to 1e-8).  At N=1 the line also carries `secondary`: configs 1 and 2 time-to-1e-8 (complete solves).

A step runs every SURVEY §8(a) row: D-update, sketch + Nystrom factorisation, PCG with the fused
matvec and preconditioner, Newton RHS / recovery, predictor-corrector, residuals/TC/PEU, initial
point, with the problem resident in HBM.  `value` = seconds per step (lower is better); `e2e` = the
same step through the C ABI with HOST buffers (H2D of A, q, b, c and D2H of x, y, z inside the
timed region).  `roofline` = the dominant kernel K1 (fused normal matvec) against the HBM copy peak;
`sketch_roofline` = the two sketch GEMMs (fp64 DMMA) against the measured DMMA peak.  Multi-GPU
(torchrun): A's columns are sharded over ranks; timing is on the device, max over ranks.
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
# (profiles/, per config and shape); None until captured for that config
#   config 4 slice (m = n = 50000): 20.000958 GB read + 4.215 MB written, profiles/r02_matvec_m50000_full.ncu-rep
TRAFFIC = {1: 134.6e6, 4: 20.000958e9 + 4.214784e6}
# read-only stream ceiling on this pool's B200 (tools/hbm_sustained.py: torch.sum over 4 GB, burst 6863 GB/s,
# sustained 6828 GB/s at full clocks; the read+write copy of MEASURED_PEAKS.json sustains 6520): K1 reads A
# once and writes only partial rows, so it can exceed the copy figure
READ_STREAM_GBS = 6863.0
# fp64 tensor-core (DMMA, mma.sync.f64) peak measured on this pool's B200 by tools/dmma_probe.cu
# (profiles/r01_dmma_peak_probe.log: 36.8-37.1 TFLOP/s over shapes / warps; cuBLAS square DGEMM 36.2)
DMMA_PEAK_TFLOPS = 37.1
# persistent PCG kernel, dram__bytes_read.sum + dram__bytes_write.sum per ITERATION (ncu --set full of
# a 20-iteration launch, config 1: 2.535 GB + 20.9 MB; profiles/r01_pcg_persistent_cfg1_20it_full.ncu-rep)
# measured DRAM bytes (read + write) per PCG iteration of the persistent kernels: config 1
# profiles/r01_pcg_persistent_cfg1_20it_final_full.ncu-rep; config-4 slice (key (4, columns per GPU))
# profiles/r02_ncu_pcg_cluster_cfg4_summary.txt (8 iterations: 160.20 GB read + 69.9 MB written)
PCG_TRAFFIC_PER_IT = {1: 85.6e6, (4, 50000): 20.034e9}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def host_info():
    """lscpu model, logical cores and host RAM (recorded with every CPU number)."""
    info = {"cores": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
            elif line.startswith("Socket(s):"):
                info["sockets"] = int(line.split(":", 1)[1])
    except Exception:
        pass
    try:
        import psutil
        info["ram_gb"] = round(psutil.virtual_memory().total / 2**30, 1)
    except Exception:
        pass
    try:
        import numpy as np
        cfg = np.show_config(mode="dicts")
        info["blas"] = cfg["Build Dependencies"]["blas"]["name"] + " " + str(cfg["Build Dependencies"]["blas"].get("version", ""))
    except Exception:
        pass
    return info


class ClockSampler:
    """Clocks / throttle reasons sampled DURING the timed region, as the profiling recipe does: ONE
    `nvidia-smi --query-gpu=... -lms 200` process started before the warm-up (its NVML start-up stays
    out of the timed region; an nvidia-smi process spawned per sample stalled the short solves' host
    calls: config 3 measured 41.6 vs 30.9 ms per solve) and stopped after; a reader thread stamps each
    line, and summary() keeps the lines that arrived between mark_start() and mark_end()."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int = 0):
        self.gpu = gpu
        self.lines = []
        self.t0 = self.t1 = None
        self._p = None
        self._t = None

    def start(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._p = None
            return self

        def reader():
            for line in self._p.stdout:
                self.lines.append((time.time(), [x.strip() for x in line.strip().split(",")]))
        self._t = threading.Thread(target=reader, daemon=True)
        self._t.start()
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time() + 0.25   # the sample that was being taken at the end
        time.sleep(0.3)

    def stop(self):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
        if self._t is not None:
            self._t.join(timeout=5)

    def summary(self):
        import statistics
        samples = [f for t, f in self.lines if self.t0 is not None and self.t0 <= t <= (self.t1 or t)]
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(x[0]) for x in samples if x[0].replace(".", "").isdigit()]
        mx = [float(x[1]) for x in samples if len(x) > 1 and x[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for x in samples for k in range(4) if len(x) > 3 + k and x[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(samples), "sampler": "nvidia-smi -lms 200 (one process)"}


# ------------------------------------------------------------------------------------------------
# workloads
# ------------------------------------------------------------------------------------------------
def cfg4_name(n_per_gpu: int, world: int) -> str:
    n = n_per_gpu * world
    return (f"cfg4_large_m50000_l200_{n_per_gpu}cols_per_gpu" + ("_slice_A25" if world == 1 and n < 400000 else "")
            + ("_full_n400000" if n == 400000 else ""))


class Workload:
    """This rank's share of one BASELINE config, resident on the device, plus what the e2e leg
    and the CPU baseline need.  Input generation only (synth/); no method arithmetic here."""

    def __init__(self, cfg: int, rank: int, world: int, device, n_per_gpu: int, dist=None):
        import numpy as np
        import torch
        self.cfg = cfg
        self.structure = 0
        self.unit_blocks = None
        self.inst = None
        dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
        if cfg == 4:
            from synth import large
            n = n_per_gpu * world
            lo, hi = large.shard_bounds(n, rank, world)
            sh = large.generate_shard(large.FULL_M, n, lo, hi, n_gen=large.FULL_N, device=device)
            b = sh.b_part
            if world > 1:
                dist.all_reduce(b)
            self.m, self.n, self.lo, self.hi, self.ell = large.FULL_M, n, lo, hi, large.ELL
            self.At, self.lda, self.q, self.b, self.c = sh.At, sh.lda, sh.q, b, sh.c
            self.name = cfg4_name(n_per_gpu, world)
            self.scaling = "weak"
            return
        from paper_2404_14524_b200 import colmajor_device
        from synth import make_config
        inst = make_config(cfg)
        self.inst = inst
        self.m, self.ell, self.name = inst.m, inst.ell, inst.name
        self.scaling = "strong"
        if cfg == 2:
            # SVM-structured A = [Xt, -Xt, I, -I]: the dense block Xt is the operand.
            # Multi-GPU: rank g holds feature columns Xt[:, f_g] (its w+ / w- variables) and the xi / s
            # variables of one row range (one unit block); e and the A u partials are all-reduced.
            Xt = inst.extra["Xt"]
            N, dd = Xt.shape
            self.structure = 1
            f0, f1 = (dd * rank) // world, (dd * (rank + 1)) // world
            r0, r1 = (N * rank) // world, (N * (rank + 1)) // world
            idx = np.concatenate([np.arange(f0, f1), dd + np.arange(f0, f1), 2 * dd + np.arange(r0, r1),
                                  2 * dd + N + np.arange(r0, r1)])
            self.n, self.lo, self.hi = inst.n, 0, len(idx)
            self.unit_blocks = [(r0, r1 - r0, 1.0)]
            self.At, self.lda = colmajor_device(np.asfortranarray(Xt[:, f0:f1]), device=device)
            self.q, self.b, self.c = dv(inst.q[idx]), dv(inst.b), dv(inst.c[idx])
            self.A_dense_block = Xt
            return
        n = inst.n
        self.n = n
        self.lo, self.hi = (n * rank) // world, (n * (rank + 1)) // world
        self.At, self.lda = colmajor_device(np.asfortranarray(inst.A[:, self.lo:self.hi]), device=device)
        self.q, self.b, self.c = dv(inst.q[self.lo:self.hi]), dv(inst.b), dv(inst.c[self.lo:self.hi])

    @property
    def ncols(self):
        return self.At.shape[0]

    def a_bytes(self):
        return 8.0 * self.m * self.ncols


# config-4 slice step (3 outer iterations) as measured on the GPU (profiles/r02_bench_cfg4_slice_final5.json):
# 124 PCG iterations incl. the initial point's 2 solves = 124 operator applications, plus per outer
# iteration ~3 operator-equivalents of N-only / T-only passes (xi, recovery x2, residuals) and 2 at the
# initial point; 4 sketches + Nystrom factorisations (initial point + 3 outer iterations).
CFG4_STEP_COUNTS = {"matvecs": 124 + 3 * 3 + 2, "sketches": 4}


def run_reference(args):
    """--impl reference: the CPU oracle (numpy/scipy fp64, oracle/) as it stands, on this host's cores.

    configs 0/1/3: each step is one complete oracle Nys-IP-PMM solve (path K) of the same instance.
    configs 2/4: the oracle cannot finish the step in minutes (config 4: 20 GB A, each operator
    application streams it on the host); each step times a bounded sample of the same workload — the
    oracle's normal matvec and its sketch + Nystrom factorisation on a column sample — and projects it to
    the step's operator-application and sketch counts.  W + K steps run, like the GPU arm."""
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    hi = host_info()
    K, W = max(1, args.steps), max(0, args.warmup)
    times = []
    if args.config in (0, 1, 3):
        from oracle import ippmm
        from synth import make_config
        inst = make_config(args.config)
        res = None
        for i in range(W + K):
            t0 = time.perf_counter()
            res = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell))
            if i >= W:
                times.append(time.perf_counter() - t0)
        sample = (f"one complete oracle Nys-IP-PMM solve of {inst.name} to 1e-8 per step ({res.outer} outer / "
                  f"{res.inner_total} PCG iterations)")
        config = {"workload": inst.name, "m": inst.m, "n": inst.n, "ell": inst.ell, "tol": 1e-8,
                  "step": "solve to 1e-8"}
    else:
        n = args.n_per_gpu * max(1, args.gpus)
        prep = cpu_projection_prepare(args.config, n)
        proj = None
        for i in range(W + K):
            if args.config == 4:
                proj = cpu_projection_step(prep, matvecs=CFG4_STEP_COUNTS["matvecs"], sketches=CFG4_STEP_COUNTS["sketches"])
            else:   # config 2 to 1e-8: the GPU solve's counts (19 outer, ~22900 PCG iterations, profiles/r01_bench_cfg2_s6.json)
                proj = cpu_projection_step(prep, matvecs=22862 + 19 * 3 + 2, sketches=20)
            if i >= W:
                times.append(proj["value"])
        sample = proj["sample"]
        config = {"workload": cfg4_name(args.n_per_gpu, max(1, args.gpus)) if args.config == 4 else prep["workload"],
                  "m": prep["m"], "n": n, "ell": prep["ell"], "tol": 1e-8,
                  "step": (f"{args.max_outer if args.max_outer is not None else 3} outer iterations"
                           if args.config == 4 else "solve to 1e-8")}
    v = float(np.mean(times))
    line = {"metric": METRIC, "value": v, "unit": "s", "impl": "reference", "n_gpus": args.gpus, "steps": K,
            "warmup": W, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "weak" if args.config == 4 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
            "cpu_baseline": {"value": v, "unit": "s", "cores": hi.get("cores"), "kind": "oracle", "sample": sample,
                             "host": hi},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_projection_prepare(cfg: int, n: int, cols: int = 1000):
    """A column sample of the config's A (the same instance recipe), resident on the host."""
    import numpy as np
    if cfg == 4:
        from synth import large
        sh = large.generate_shard(large.FULL_M, n, 0, cols, n_gen=large.FULL_N, device="cpu")
        A = np.asfortranarray(sh.At[:, :large.FULL_M].numpy().T)
        return {"A": A, "e": None, "m": large.FULL_M, "ell": large.ELL, "scale": n / cols,
                "workload": f"cfg4 m=50000 n={n} l=200"}
    from synth import make_config
    inst = make_config(cfg)
    A = inst.extra["Xt"] if cfg == 2 else inst.A
    return {"A": A, "e": np.ones(inst.m) if cfg == 2 else None, "m": inst.m, "ell": inst.ell, "scale": 1.0,
            "workload": inst.name}


def cpu_projection_step(prep, matvecs: int, sketches: int):
    """Oracle time for one step projected from a bounded sample (a few s of CPU work): the oracle's
    normal matvec and its sketch + Nystrom factorisation timed on the column sample, scaled by
    (total columns / sample columns) and by the step's operator-application / sketch counts."""
    import numpy as np
    from oracle import linops, nystrom
    from oracle.rng import gaussian_omega
    A, e, m, ell, scale = prep["A"], prep["e"], prep["m"], prep["ell"], prep["scale"]
    rs = np.random.default_rng(0)
    d = rs.uniform(0.1, 2.0, A.shape[1])
    v = rs.standard_normal(m)
    t0 = time.perf_counter()
    linops.normal_matvec(A, d, v, 1e-3, e)
    t_mv = (time.perf_counter() - t0) * scale
    Om = gaussian_omega(m, ell, 0, 1)
    t0 = time.perf_counter()
    Y = linops.sketch(A, d, Om, e)
    t_sk = (time.perf_counter() - t0) * scale
    t0 = time.perf_counter()
    nystrom.nystrom_from_sketch(Y * scale, Om)
    t_fac = time.perf_counter() - t0
    value = matvecs * t_mv + sketches * (t_sk + t_fac)
    sample = (f"oracle normal matvec and sketch+Nystrom on {A.shape[1]} of {int(round(A.shape[1] * scale))} columns of "
              f"{prep['workload']}: {t_mv:.3g} s/matvec, {t_sk + t_fac:.3g} s/sketch at full size; projected to "
              f"{matvecs} operator applications + {sketches} sketches per step")
    return {"value": value, "sample": sample, "workload": prep["workload"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n-per-gpu", type=int, default=50000, help="config 4: columns of A per rank")
    ap.add_argument("--prec-refresh", type=int, default=1,
                    help="SURVEY §8(f) f3: rebuild the Nystrom preconditioner every K outer iterations (1 = Alg. 3)")
    ap.add_argument("--precond", default="nystrom", choices=["nystrom", "chol"],
                    help="nystrom: Nys-IP-PMM (default); chol: Chol-IP-PMM, partial Cholesky of rank ell (f2)")
    ap.add_argument("--prec-growth", type=float, default=0.0,
                    help="f3: also rebuild when PCG counts grow by this factor since the last rebuild (0 = off)")
    ap.add_argument("--ell-max", type=int, default=0,
                    help="f3 adaptive rank (reading F1): double ell up to this cap while lam_hat_ell > 10 delta (0 = off)")
    ap.add_argument("--max-outer", type=int, default=None,
                    help="cap on IP-PMM outer iterations (default: 3 for config 4, 100 otherwise); below 100 the "
                         "step is 'max-outer iterations', not time-to-1e-8 (config 4's one-GPU slice is "
                         "ill-conditioned: DESIGN.md §2, A25)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the configs 1 and 2 time-to-1e-8 legs of the N=1 line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--matvec-reps", type=int, default=50)
    args = ap.parse_args()
    if args.max_outer is None:
        args.max_outer = 3 if args.config == 4 else 100
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2404_14524_b200 import Context, nccl_unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    else:
        nid = None
    stream = torch.cuda.Stream(local)
    ctx = Context(local, stream=stream, nccl_id=nid, rank=rank, world=world)

    wl = Workload(args.config, rank, world, device, args.n_per_gpu, dist if world > 1 else None)
    torch.cuda.synchronize()
    m, nloc, lda = wl.m, wl.ncols, wl.lda

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def one_solve():
        with torch.cuda.stream(stream):
            return ctx.nys_ipppmm_solve(wl.At, lda, m, wl.q, wl.b, wl.c, ell=wl.ell, structure=wl.structure,
                                        unit_blocks=wl.unit_blocks, prec_refresh=args.prec_refresh, prec_growth=args.prec_growth,
                                        precond=1 if args.precond == "chol" else 0, ell_max=args.ell_max,
                                        max_outer=args.max_outer)

    # ---- secondary legs (N = 1, headline run only): configs 1 and 2 time-to-1e-8, complete solves ------
    # run BEFORE the headline: the 20 GB headline step drives the GPU into its power cap (SM clock
    # ~1650-1870 MHz), and the short config-1 solves measured right after it ran ~15 % slower (95.7 vs
    # 82.8 ms on one box) than on a GPU that was not just throttled
    secondary = None
    if world == 1 and args.config == 4 and not args.no_secondary:
        secondary = {}
        for sc in (1, 2):
            w2 = Workload(sc, 0, 1, device, 0)

            def solve2(w2=w2):
                with torch.cuda.stream(stream):
                    return ctx.nys_ipppmm_solve(w2.At, w2.lda, w2.m, w2.q, w2.b, w2.c, ell=w2.ell,
                                                structure=w2.structure, unit_blocks=w2.unit_blocks)
            for _ in range(3):
                solve2()
            barrier()
            K2 = 3
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r2 = [solve2() for _ in range(K2)]
            e1.record(stream)
            barrier()
            g2 = r2[-1]
            secondary[f"config{sc}"] = {
                "workload": w2.name, "metric": "Nys-IP-PMM time-to-1e-8", "value": e0.elapsed_time(e1) / 1e3 / K2,
                "unit": "s", "steps": K2, "warmup": 3, "status": g2["status"], "outer": g2["outer"],
                "inner": g2["inner"], "obj": g2["obj"], "rel_p": g2["rel_p"], "rel_d": g2["rel_d"], "mu": g2["mu"],
                "t_sketch_ms": g2["t_sketch_ms"], "t_pcg_ms": g2["t_pcg_ms"], "t_other_ms": g2["t_other_ms"]}
            del w2, r2
            torch.cuda.empty_cache()

    # ---- warm-up ------------------------------------------------------------------------------
    clk = ClockSampler(local).start()
    W = max(args.warmup, 3)
    for _ in range(W):
        g = one_solve()
    assert g["status"] == 0 or (args.max_outer < 100 and g["status"] == -5), f"solve status {g['status']}"
    # ---- timed region: K complete solves, CUDA events on the library's stream ------------------
    barrier()
    launches0 = ctx.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark_start()
    ev0.record(stream)
    results = [one_solve() for _ in range(args.steps)]
    ev1.record(stream)
    barrier()
    clk.mark_end()
    clk.stop()
    launches = ctx.kernel_launches - launches0
    t_dev = ev0.elapsed_time(ev1) / 1e3
    if world > 1:
        tt = torch.tensor([t_dev], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
    sec_per_solve = t_dev / args.steps
    last = results[-1]
    matvecs_per_solve = last["matvecs"]

    # ---- dominant kernel: fused normal matvec, timed live with CUDA events on its stream ------
    # Launches captured in CUDA graphs (no host gaps).  If A fits in L2 (< 1 GB), each launch is
    # preceded by a 256 MB L2-flushing read and that read's own time is subtracted; otherwise
    # A itself is larger than L2 and the launches are back to back.
    rs = np.random.default_rng(0)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
    d = dv(rs.uniform(0.01, 2.0, nloc))
    v = dv(rs.standard_normal(m))
    w = torch.empty(m, dtype=torch.float64, device=device)
    e_diag = dv(np.ones(m)) if wl.structure == 1 else None
    small = wl.a_bytes() < 1e9
    R = args.matvec_reps if small else max(6, min(args.matvec_reps, int(1.2e11 / wl.a_bytes())))
    flush = torch.ones(32 * 1024 * 1024, dtype=torch.float64, device=device) if small else None
    fl_out = torch.empty((), dtype=torch.float64, device=device)

    def mv():
        ctx.nys_normal_matvec(wl.At, lda, m, d, e_diag, 1e-3, v, w)

    def fl():
        torch.sum(flush, dim=0, out=fl_out)

    with torch.cuda.stream(stream):
        for _ in range(3):
            mv()
    barrier()

    def capture(fn):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            for _ in range(R):
                fn()
        return gr

    def timed(gr):
        gr.replay()
        barrier()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        with torch.cuda.stream(stream):
            gr.replay()
        b_.record(stream)
        barrier()
        return a.elapsed_time(b_) / 1e3

    g_warm = capture(mv)
    mv_warm_s = sorted(timed(g_warm) for _ in range(3))[1] / R     # median of 3 graph replays
    if small:
        g_cold = capture(lambda: (fl(), mv()))
        g_flush = capture(fl)
        mv_s = (timed(g_cold) - timed(g_flush)) / R
        del g_cold, g_flush
    else:
        mv_s = mv_warm_s
    del g_warm, flush
    mv_bytes = 8.0 * (m * nloc + nloc + 2 * m)  # A once + d + v in + w out
    mv_gbs = mv_bytes / mv_s / 1e9
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"

    # ---- persistent PCG kernel (single GPU): ONE launch per PCG solve, the dominant kernel of the step
    # (m <= 8192: pcg_persistent_kernel; m > 8192: pcg_cluster_kernel, k_pcgc.cu).  Timed live:
    # nys_pcg_solve with tol = 0 runs exactly I iterations; two calls (I1 < I2 iterations) are differenced,
    # so the call's setup kernels and its true-residual matvec cancel and t_it is the kernel's own time
    # per iteration (the launch's one-off pipeline fill, ~10 us, is spread over I2 - I1 iterations)
    pcg_roof = None
    if world == 1 and m <= 16 * 8640 and wl.structure == 0 and 0 < wl.ell <= 256:
        ell = wl.ell
        mp = m + (m % 2)
        Om = torch.empty((ell, mp), dtype=torch.float64, device=device)
        U = torch.empty((ell, mp), dtype=torch.float64, device=device)
        lam = torch.empty(ell, dtype=torch.float64, device=device)
        rhs = dv(rs.standard_normal(m))
        xs = torch.zeros(m, dtype=torch.float64, device=device)
        I2 = 400 if small else max(20, min(400, int(8e11 / wl.a_bytes())))
        with torch.cuda.stream(stream):
            ctx.nys_gaussian(m, ell, 0, 1, Om)
            ctx.nys_sketch(wl.At, lda, m, d, None, 1e-2, ell, Om, U, lam)
            ctx.nys_pcg_solve(wl.At, lda, m, d, None, 1e-2, ell, U, lam, 1e-2, rhs, xs, 0.0, 4)
        barrier()
        from paper_2404_14524_b200 import NysError

        def pcg_call(iters):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            xs.zero_()
            barrier()
            a_.record(stream)
            with torch.cuda.stream(stream):
                inf = ctx.nys_pcg_solve(wl.At, lda, m, d, None, 1e-2, ell, U, lam, 1e-2, rhs, xs, 0.0, iters)
            b_.record(stream)
            barrier()
            return inf, a_.elapsed_time(b_) / 1e3

        while True:
            # at small m, I2 iterations run far past convergence; once r reaches the rounding floor
            # p^T N p can lose its sign (EBREAKDOWN): time fewer iterations then
            try:
                I1 = max(2, I2 // 4)
                info1, t1 = pcg_call(I1)
                info, t2 = pcg_call(I2)
            except NysError:
                if I2 <= 25:
                    raise
                I2 //= 2
                continue
            break
        if info.iters - info1.iters >= 2:
            t_it = (t2 - t1) / (info.iters - info1.iters)
            timing = (f"two launches of {info1.iters} and {info.iters} iterations differenced (setup and the "
                      "call's true-residual matvec cancel)")
        else:   # the solve reaches the rounding floor (r = 0) within I1 iterations (config 3: l = m)
            t_it = t2 / max(1, info.iters)
            timing = f"one launch of {info.iters} iterations (the call's setup and true-residual matvec included)"
        t_call = t2
        # SURVEY §8(d) per CG iteration: one K1 + 16 m l bytes of U (U^T r and U h) + ~10 m-vectors
        it_bytes = mv_bytes + 16.0 * m * ell + 80.0 * m
        pcg_gbs = it_bytes / t_it / 1e9
        key = (args.config, wl.ncols) if args.config == 4 else args.config
        tr_it = PCG_TRAFFIC_PER_IT.get(key)
        pcg_roof = {"bound": "hbm", "achieved": pcg_gbs, "peak": hbm, "unit": "GB/s", "frac": pcg_gbs / hbm,
                    # measured DRAM bytes (ncu) per iteration x the iterations of one launch
                    "traffic": tr_it * info.iters if tr_it else None,
                    # at config 1 A (128 MB) is about the L2 size: part of it survives in L2 between
                    # iterations, so DRAM traffic < algorithmic bytes; frac above is the effective
                    # ALGORITHMIC bandwidth, dram_frac the measured-DRAM-bytes one
                    "dram_frac": (tr_it / t_it / 1e9 / hbm) if tr_it else None,
                    "kernel": ("pcg_persistent_kernel" if m <= 8192 else "pcg_cluster_kernel (k_pcgc.cu)")
                              + ": the whole PCG solve in one cooperative launch",
                    "peak_source": peak_src, "iterations_per_launch": info.iters,
                    "bytes_per_iteration": it_bytes, "bytes_per_launch": info.iters * it_bytes,
                    "launch_us": t_call * 1e6, "us_per_iteration": t_it * 1e6,
                    "timing": timing,
                    "share_of_step": (last["t_pcg_ms"] / 1e3) / sec_per_solve}

    # ---- sketch GEMMs (K2 + K3, fp64 DMMA): Y = A (d o (A^T Omega)), 4 m n l flops per call (SURVEY
    # §8(d)), timed live with CUDA events on the library stream (the sketch is a dense contraction: its
    # roofline is the fp64 tensor pipe, DMMA_PEAK_TFLOPS measured by tools/dmma_probe.cu)
    sk_roof = None
    if wl.ell > 0 and wl.structure == 0 and nloc > 0:
        ell = wl.ell
        mp = m + (m % 2)
        Om_s = torch.empty((ell, mp), dtype=torch.float64, device=device)
        Y_s = torch.empty((ell, mp), dtype=torch.float64, device=device)
        with torch.cuda.stream(stream):
            ctx.nys_gaussian(m, ell, 0, 1, Om_s)
            ctx.nys_sketch_apply(wl.At, lda, m, d, None, ell, Om_s, Y_s)
        barrier()
        RS = 3 if wl.a_bytes() > 1e9 else 20
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(RS):
                ctx.nys_sketch_apply(wl.At, lda, m, d, None, ell, Om_s, Y_s)
        b_.record(stream)
        barrier()
        t_sk = a_.elapsed_time(b_) / 1e3 / RS
        if world > 1:
            tt = torch.tensor([t_sk], device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_sk = float(tt.item())
        sk_flops = 4.0 * m * nloc * ell
        sk_tf = sk_flops / t_sk / 1e12
        sk_roof = {"bound": "tensor", "achieved": sk_tf, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                   "frac": sk_tf / DMMA_PEAK_TFLOPS, "traffic": None,
                   "kernel": "sketch Y = A (d o (A^T Omega)): two fp64 DMMA GEMMs (mma.sync.f64), nys_sketch_apply",
                   "peak_source": "measured fp64 DMMA peak, tools/dmma_probe.cu, profiles/r01_dmma_peak_probe.log "
                                  "(MEASURED_PEAKS.json has no fp64 entry)",
                   "flops_per_call": sk_flops, "call_us": t_sk * 1e6,
                   "share_of_step": (last["outer"] + 1) * t_sk / sec_per_solve if args.ell_max == 0 else None}
        del Om_s, Y_s

    # ---- e2e: the same solve through the C ABI with host buffers --------------------------------
    e2e = None
    if not args.no_e2e:
        need = wl.a_bytes() * 1.2
        try:
            import psutil
            avail = psutil.virtual_memory().available / max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
        except Exception:
            avail = float("inf")
        if need < 0.6 * avail:
            # inputs in PINNED host memory (the contract's H2D leg), copied in by the library each step
            def pinned(t):
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t)
                return h
            A_pin, q_pin, b_pin, c_pin = pinned(wl.At), pinned(wl.q), pinned(wl.b), pinned(wl.c)
            A_host, qh, bh, ch = A_pin.numpy(), q_pin.numpy(), b_pin.numpy(), c_pin.numpy()
            with torch.cuda.stream(stream):  # one untimed e2e solve: workspace for the host path, graphs
                ctx.nys_ipppmm_solve(A_host, lda, m, qh, bh, ch, ell=wl.ell, host=True, structure=wl.structure,
                                     unit_blocks=wl.unit_blocks, prec_refresh=args.prec_refresh, prec_growth=args.prec_growth,
                                     precond=1 if args.precond == "chol" else 0, ell_max=args.ell_max,
                                        max_outer=args.max_outer)
            barrier()
            t0 = time.perf_counter()
            E_STEPS = max(1, min(args.steps, 3))
            for _ in range(E_STEPS):
                with torch.cuda.stream(stream):
                    ctx.nys_ipppmm_solve(A_host, lda, m, qh, bh, ch, ell=wl.ell, host=True, structure=wl.structure,
                                         unit_blocks=wl.unit_blocks, prec_refresh=args.prec_refresh, prec_growth=args.prec_growth,
                                         precond=1 if args.precond == "chol" else 0, ell_max=args.ell_max,
                                        max_outer=args.max_outer)
            barrier()
            t_e2e = (time.perf_counter() - t0) / E_STEPS
            if world > 1:
                tt = torch.tensor([t_e2e], device=device)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_e2e = float(tt.item())
            nq = qh.shape[0]
            e2e = {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": int(A_host.nbytes + 8 * (2 * nq + m)),
                   "d2h_bytes_per_step": int(8 * (2 * nq + m)), "host_buffers": "pinned"}
            del A_host, A_pin
        else:
            e2e = {"value": None, "unit": "s", "skipped": f"host RAM: need {need / 1e9:.0f} GB pinned-able, "
                                                          f"{avail / 1e9:.0f} GB available per rank"}

    # ---- CPU oracle baseline (rank 0, N = 1 only; bounded sample) --------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.config in (0, 1, 3):
            from oracle import ippmm
            inst = wl.inst
            t0 = time.perf_counter()
            r = ippmm.solve(inst.A, inst.q, inst.b, inst.c, ippmm.Options(path="krylov", ell=inst.ell))
            tc = time.perf_counter() - t0
            cpu = {"value": tc, "unit": "s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"one full oracle solve of {inst.name} ({r.outer} outer, {r.inner_total} PCG iters, "
                             f"obj {r.obj:.12g} vs GPU {last['obj']:.12g})"}
        else:
            prep = cpu_projection_prepare(args.config, wl.n)
            proj = cpu_projection_step(prep, matvecs=matvecs_per_solve + 3 * last["outer"] + 2,
                                       sketches=last["outer"] + 1)
            cpu = {"value": proj["value"], "unit": "s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": proj["sample"]}
            del prep
        cpu["host"] = host_info()

    mv_roof = {"bound": "hbm", "achieved": mv_gbs, "peak": hbm, "unit": "GB/s", "frac": mv_gbs / hbm,
               "traffic": TRAFFIC.get(args.config) if (args.config != 4 or (wl.ncols == 50000 and world == 1)) else None,
               "kernel": "fused normal matvec K1 standalone (matvec_kernel + mv_finalize, nys_normal_matvec, "
                         "graph-captured): the streaming pipeline of the PCG kernels' matvec phase and of the "
                         "T / N / BOTH passes",
               "peak_source": peak_src, "bytes_per_launch": mv_bytes, "launch_us": mv_s * 1e6,
               "warm_l2_gbs": mv_bytes / mv_warm_s / 1e9,
               "frac_of_read_stream": mv_gbs / READ_STREAM_GBS,
               "pcg_effective_gbs": (last["inner"] * mv_bytes / (last["t_pcg_ms"] / 1e3) / 1e9) if last["t_pcg_ms"] > 0 else None,
               # the step's PCG matvecs run inside the persistent PCG kernel (roofline above) when it exists
               "share_of_step": None if pcg_roof is not None else matvecs_per_solve * mv_s / sec_per_solve}
    if rank == 0:
        line = {
            "metric": METRIC, "value": sec_per_solve, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": W, "ms_per_step": sec_per_solve * 1e3, "higher_is_better": False,
            "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name, "m": m, "n": wl.n, "ell": wl.ell, "tol": 1e-8,
                       "prec_refresh": args.prec_refresh, "prec_growth": args.prec_growth, "precond": args.precond,
                       "ell_max": args.ell_max, "max_outer": args.max_outer,
                       "step": "solve to 1e-8" if args.max_outer >= 100 else f"{args.max_outer} outer iterations",
                       "parallelism": f"column-shard x{world}",
                       "l2": (("A = %.0f MB vs 126 MB L2: the persistent-PCG roofline launch is NOT flushed (A partly "
                               "L2-resident across iterations: see roofline.dram_frac); the matvec leg is L2-flushed "
                               "(256 MB read) before each launch" % (wl.a_bytes() * world / 1e6)) if pcg_roof is not None else
                              ("A = %.0f MB vs 126 MB L2: roofline launches L2-flushed (256 MB read) before each"
                               % (wl.a_bytes() * world / 1e6))) if small else
                             ("inputs larger than L2: A = %.1f GB per GPU >> 126 MB L2 (streamed with L2 evict_first); "
                              "no flush needed" % (wl.a_bytes() / 1e9))},
            "clocks": clk.summary(),
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": pcg_roof if pcg_roof is not None else mv_roof,
            "matvec": mv_roof,
            "sketch_roofline": sk_roof,
            "secondary": secondary,
            "solve": {"outer": last["outer"], "inner": last["inner"], "obj": last["obj"], "rel_p": last["rel_p"],
                      "rel_d": last["rel_d"], "mu": last["mu"], "matvecs": matvecs_per_solve,
                      "t_sketch_ms": last["t_sketch_ms"], "t_pcg_ms": last["t_pcg_ms"],
                      "t_other_ms": last["t_other_ms"], "kernel_launches": last["kernel_launches"],
                      # PCG iterations (predictor, corrector) per outer iteration; the rest of "inner"
                      # is the initial point's two solves (App. B.2, reading A14'')
                      "pcg_per_outer": [[r["pcg_pred"], r["pcg_corr"]] for r in last.get("log", [])]},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
