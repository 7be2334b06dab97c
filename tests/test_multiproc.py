"""N > 1 path on CPU: world_size-2 `gloo` process groups.

The library shards A by columns; every m-space quantity is replicated and the only exchanges are
sums (C1: the m-vector of each normal matvec, C2: the m x l sketch, C3/C4: scalars) and mins
(ratio tests).  These tests check that decomposition on the oracle's operator and on the config-4
shard generator with a real 2-process group, and the bench's multi-rank launch contract
(rank 0 alone prints; the other ranks exit 0).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = {}
    try:
        for _ in range(world):  # drain BEFORE joining: a child blocks on exit until its put is consumed
            r, res = q.get(timeout=240)
            outs[r] = res
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert sorted(outs) == list(range(world)), outs
    return outs


def _entry(fn, rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _allreduce(a, op=dist.ReduceOp.SUM):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t, op=op)
    return t.numpy()


def _sharded_operator(rank, world):
    from oracle import linops
    from synth import make_config
    inst = make_config(1, m=300, n=1201, ell=20)
    n = inst.n
    lo, hi = (n * rank) // world, (n * (rank + 1)) // world
    rs = np.random.default_rng(7)
    d = rs.uniform(0.01, 3.0, n)
    v = rs.standard_normal(inst.m)
    Om = rs.standard_normal((inst.m, 20))
    delta = 0.25
    # C1: each rank applies its own columns (no delta), one sum, then delta v on the replicated vector
    w = _allreduce(linops.normal_matvec(inst.A[:, lo:hi], d[lo:hi], v, 0.0)) + delta * v
    # C2: the sketch
    Y = _allreduce(linops.sketch(inst.A[:, lo:hi], d[lo:hi], Om))
    # C3/C4: scalars  x^T z / n and the ratio-test min over the local slice
    x = rs.uniform(0.1, 1.0, n)
    z = rs.uniform(0.1, 1.0, n)
    dx = rs.standard_normal(n)
    mu = _allreduce(np.array([x[lo:hi] @ z[lo:hi]]))[0] / n
    neg = dx[lo:hi] < 0
    amin = np.min(-x[lo:hi][neg] / dx[lo:hi][neg]) if neg.any() else np.inf
    amin = _allreduce(np.array([amin]), op=dist.ReduceOp.MIN)[0]
    return {"w": w, "Y": Y, "mu": mu, "amin": amin, "lohi": (lo, hi)}


def test_column_sharded_operator_sketch_and_scalars_gloo():
    from oracle import linops
    from synth import make_config
    outs = _run(_sharded_operator)
    inst = make_config(1, m=300, n=1201, ell=20)
    rs = np.random.default_rng(7)
    d = rs.uniform(0.01, 3.0, inst.n)
    v = rs.standard_normal(inst.m)
    Om = rs.standard_normal((inst.m, 20))
    w_ref = linops.normal_matvec(inst.A, d, v, 0.25)
    Y_ref = linops.sketch(inst.A, d, Om)
    x = rs.uniform(0.1, 1.0, inst.n)
    z = rs.uniform(0.1, 1.0, inst.n)
    dx = rs.standard_normal(inst.n)
    neg = dx < 0
    for r in (0, 1):
        o = outs[r]
        assert np.linalg.norm(o["w"] - w_ref) <= 1e-13 * np.linalg.norm(w_ref)
        assert np.linalg.norm(o["Y"] - Y_ref) <= 1e-13 * np.linalg.norm(Y_ref)
        assert abs(o["mu"] - x @ z / inst.n) <= 1e-15 * (x @ z)
        assert o["amin"] == np.min(-x[neg] / dx[neg])
    # identical replicated results on both ranks (what keeps the ranks' scalar decisions in step)
    assert np.array_equal(outs[0]["w"], outs[1]["w"]) and np.array_equal(outs[0]["Y"], outs[1]["Y"])
    # the column partition covers [0, n) exactly once
    assert outs[0]["lohi"][0] == 0 and outs[0]["lohi"][1] == outs[1]["lohi"][0] and outs[1]["lohi"][1] == inst.n


def _config4_shards(rank, world):
    from synth import large
    m, n = 150, 999
    lo, hi = large.shard_bounds(n, rank, world)
    sh = large.generate_shard(m, n, lo, hi, n_gen=2000)
    b = torch.from_numpy(sh.b_part.numpy().copy())
    dist.all_reduce(b)
    return {"At": sh.At.numpy(), "b": b.numpy(), "c": sh.c.numpy(), "lo": lo, "hi": hi}


def test_config4_generation_is_rank_count_invariant_gloo():
    from synth import large
    outs = _run(_config4_shards)
    full = large.generate_shard(150, 999, 0, 999, n_gen=2000)
    At = np.concatenate([outs[0]["At"], outs[1]["At"]])
    assert np.array_equal(At, full.At.numpy())
    assert np.array_equal(np.concatenate([outs[0]["c"], outs[1]["c"]]), full.c.numpy())
    for r in (0, 1):
        assert np.allclose(outs[r]["b"], full.b_part.numpy(), rtol=1e-13, atol=1e-10)
    assert np.array_equal(outs[0]["b"], outs[1]["b"])


def test_bench_reference_arm_under_torchrun_rank0_only():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--config", "0",
           "--steps", "1", "--warmup", "0"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2 and rec["cpu_baseline"]["kind"] == "oracle"
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["value"] > 0
