"""Summarise an ncu report: key SOL / scheduler metrics and the SASS instruction mix (by opcode) with
stall-sample shares.  Usage: python tools/ncu_mix.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ("Duration", "DRAM Throughput", "Memory Throughput", "SM Frequency", "Issue Slots Busy", "Executed Ipc Active",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Grid Size", "Block Size")
for r in csv.reader(io.StringIO(det)):
    if len(r) > 3 and r[-3] in keys:
        print(f"  {r[-3]:40s} {r[-1]:>14s} {r[-2]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
iS, iSm, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
agg = collections.defaultdict(lambda: [0, 0])
for r in rows[2:]:
    if len(r) <= iE:
        continue
    toks = r[iS].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    agg[op.split(".")[0]][0] += int(r[iE] or 0)
    agg[op.split(".")[0]][1] += int(r[iSm] or 0)
te = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"  SASS mix ({te} warp instructions):")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:16]:
    print(f"    {k:10s} {v[0] / te:6.1%} exec  {v[1] / max(ts, 1):6.1%} stall samples")
