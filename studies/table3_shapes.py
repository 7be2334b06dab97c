"""The paper's Table 3 workloads (dual SVM of App. C.2) at their dataset SHAPES, solved to
1e-8 on one B200 through the library (structure 2: the identity block of the dual SVM is never
stored).  The data are synthetic stand-ins (synth.make_svm_dual: a two-class Gaussian mixture), so
iteration counts differ from the paper's real datasets; the paper's CPU times (16 EPYC cores, Julia)
are printed as context only.  ell follows Table 3 (capped at 256; STL-10 uses 800 in the paper).
Sparse datasets (Dexter, Sector) are out of scope (dense A only).

    python -m studies.table3_shapes [--only RNASeq,SensIT] [--arms nys,cg,chol] [--out file.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# name: (features d, instances n, ell in Table 3, paper Nys / CG / Chol seconds (None = not reported))
TABLE3 = {
    "SensIT": (100, 98528, 50, (5.69, 14.12, 11.05)),
    "CIFAR10": (3072, 60000, 200, (1103.26, None, None)),
    "RNASeq": (20531, 801, 200, (8.40, 19.59, 769.95)),
    "STL-10": (27648, 13000, 800, (7691.41, 30016.8, 103681.65)),
    "Arcene": (10000, 100, 20, (0.233, 0.278, 18.15)),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--arms", default="nys,cg,chol")
    ap.add_argument("--out", default="")
    ap.add_argument("--max-outer", type=int, default=100)
    args = ap.parse_args()
    from paper_2404_14524_b200 import Context, colmajor_device
    from synth import make_svm_dual
    names = [n for n in TABLE3 if not args.only or n in args.only.split(",")]
    arms = args.arms.split(",")
    ctx = Context(0)
    rows = []
    dev = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(dt).cuda()  # noqa: E731
    for name in names:
        d, ns, ell_p, paper = TABLE3[name]
        ell = min(ell_p, 256)
        t0 = time.time()
        inst = make_svm_dual(ns, d, ell=ell)
        B = inst.extra["B"]
        Bd, lda = colmajor_device(B)
        del B
        kw = dict(structure=2, unit_blocks=inst.extra["unit_blocks"], vtype=dev(inst.extra["vtype"], torch.int8),
                  ub=dev(inst.extra["ub"]), max_outer=args.max_outer, max_records=0)
        qd, bd, cd = dev(inst.q), dev(inst.b), dev(inst.c)
        gen_s = time.time() - t0
        for arm in arms:
            if arm == "cg":
                e, pre = 0, 0
            elif arm == "chol":
                e, pre = ell, 1
            else:
                e, pre = ell, 0
            g = ctx.nys_ipppmm_solve(Bd, lda, inst.m, qd, bd, cd, ell=e, precond=pre, **kw)   # warm (workspace)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            ev0.record()
            g = ctx.nys_ipppmm_solve(Bd, lda, inst.m, qd, bd, cd, ell=e, precond=pre, **kw)
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
            ref = paper[{"nys": 0, "cg": 1, "chol": 2}[arm]]
            row = {"dataset_shape": name, "d": d, "n_samples": ns, "m": inst.m, "n": inst.n, "arm": arm, "ell": e,
                   "status": g["status"], "outer": g["outer"], "inner": g["inner"], "seconds": ms / 1e3,
                   "t_construct_ms": g["t_sketch_ms"], "t_pcg_ms": g["t_pcg_ms"], "rel_p": g["rel_p"],
                   "rel_d": g["rel_d"], "mu": g["mu"], "paper_cpu_seconds_context": ref,
                   "dense_block_GB": 8.0 * inst.m * ns / 1e9}
            rows.append(row)
            print(f"{name:8s} {arm:4s} ell={e:3d} m={inst.m:6d}: {ms / 1e3:8.3f} s  outer {g['outer']:3d} inner "
                  f"{g['inner']:6d} (construct {g['t_sketch_ms']:8.1f} ms, pcg {g['t_pcg_ms']:9.1f} ms) status "
                  f"{g['status']}  [paper CPU: {ref} s; generated in {gen_s:.1f} s]", flush=True)
        del Bd
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"study": "Table 3 shapes (P:1014-1042), synthetic dual SVM", "rows": rows}, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
