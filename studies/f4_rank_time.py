"""§8(f) f4 / paper §5.2.3 (Fig. "rank_time"): total / preconditioner-construction /
PCG time of Nys-IP-PMM and Chol-IP-PMM as the rank ell varies, averaged over `--runs` solves
(the paper averages 4), on a synthetic RNASeq-shaped dual SVM (App. C.2; d = 20531 features,
801 samples -> normal equations 20532 x 20532), synth.make_svm_dual.  Times are the
library's own report (t_sketch_ms = construction incl. the scaling, t_pcg_ms, t_other_ms), each
solve timed with CUDA events on the library stream as a cross-check.  ell = 0 is CG-IP-PMM.

    python -m studies.f4_rank_time [--samples 801] [--d 20531] [--ells 0,10,20,50,100,200,256] [--runs 4]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=801)
    ap.add_argument("--d", type=int, default=20531)
    ap.add_argument("--ells", default="0,10,20,50,100,200,256")
    ap.add_argument("--chol-ells", default="10,20,50,100,200,256")
    ap.add_argument("--runs", type=int, default=4)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2404_14524_b200 import Context, colmajor_device
    from synth import make_svm_dual
    inst = make_svm_dual(args.samples, args.d)
    dev = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(dt).cuda()  # noqa: E731
    B = inst.extra["B"]
    m = B.shape[0]
    Bd, lda = colmajor_device(B)
    ctx = Context(0)
    st = torch.cuda.Stream()
    kw = dict(structure=2, unit_blocks=inst.extra["unit_blocks"], vtype=dev(inst.extra["vtype"], torch.int8),
              ub=dev(inst.extra["ub"]))
    qd, bd, cd = dev(inst.q), dev(inst.b), dev(inst.c)
    torch.cuda.synchronize()
    rows = []

    def run(ell, precond):
        res = []
        for r in range(args.runs + 1):                                # first run = warm-up (workspace, graphs)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            ev0.record(torch.cuda.current_stream())
            g = ctx.nys_ipppmm_solve(Bd, lda, m, qd, bd, cd, ell=ell, seed=r, precond=precond, max_records=0, **kw)
            ev1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            if r == 0:
                continue
            res.append({"status": g["status"], "outer": g["outer"], "inner": g["inner"],
                        "total_ms": g["t_total_ms"], "construct_ms": g["t_sketch_ms"], "pcg_ms": g["t_pcg_ms"],
                        "other_ms": g["t_other_ms"], "event_ms": ev0.elapsed_time(ev1)})
        avg = {k: float(np.mean([x[k] for x in res])) for k in ("outer", "inner", "total_ms", "construct_ms",
                                                                  "pcg_ms", "other_ms")}
        avg.update({"ell": ell, "precond": "chol" if precond else ("nystrom" if ell else "none (CG-IP-PMM)"),
                    "status": [x["status"] for x in res], "runs": len(res)})
        print(f"{avg['precond']:>17s} ell={ell:3d}: total {avg['total_ms']:9.1f} ms  construct "
              f"{avg['construct_ms']:8.1f}  pcg {avg['pcg_ms']:9.1f} ({100 * avg['pcg_ms'] / avg['total_ms']:4.1f} %)  "
              f"other {avg['other_ms']:7.1f}  outer {avg['outer']:.1f} inner {avg['inner']:.0f}", flush=True)
        rows.append(avg)

    for ell in [int(v) for v in args.ells.split(",")]:
        run(ell, 0)
    for ell in [int(v) for v in args.chol_ells.split(",") if v]:
        run(ell, 1)
    out = {"study": "f4 rank vs time (P:1089-1114)", "workload": inst.name, "m": m, "n": inst.n, "rows": rows,
           "when": time.strftime("%Y-%m-%d %H:%M:%S")}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
