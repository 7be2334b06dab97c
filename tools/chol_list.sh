# per-kernel device times (ncu launch list) of one nys_sketch at each shape: the Cholesky / Jacobi kernels
for sh in "$@"; do
  python tools/sketch_bench.py $sh 1 > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cl.csv python tools/sketch_bench.py $sh 1 > /dev/null 2>&1
  python - "$sh" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open("gpurun_out/cl.csv")) if len(r) > 10]
h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
seq = [(r[ik].split("(")[0], float(r[iv]) / 1e3) for r in rows[1:]]
last = seq[len(seq) // 2:]   # the second half: the last nys_sketch call
agg = collections.defaultdict(list)
for k, v in last: agg[k].append(v)
print(sys.argv[1], "; ".join(f"{k.replace('void ', '').replace('nys::', '')} {len(v)}x{sum(v)/len(v):.1f}us" for k, v in agg.items() if "chol" in k or "jacobi" in k or "trmm" in k))
PY
done
