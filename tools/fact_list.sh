# per-kernel device times of one nys_sketch (sketch + Nystrom factorisation) at each shape (ncu launch list)
for sh in "$@"; do
  python tools/sketch_bench.py $sh 1 > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fl.csv python tools/sketch_bench.py $sh 1 > /dev/null 2>&1
  python - "$sh" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/fl.csv")) if len(r) > 10]
h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
seq = [(r[ik].split("(")[0].replace("void ", "").replace("nys::", ""), float(r[iv]) / 1e3) for r in rows[1:]]
# the last nys_sketch call: from the last gaussian-free sketch GEMM pair to the end
print("==", sys.argv[1], "kernels:", len(seq))
tail = seq[-40:]
tot = 0.0
for k, v in tail:
    tot += v
    print(f"  {v:8.1f} us  {k[:70]}")
print(f"  total of the last 40: {tot:.1f} us")
PY
done
