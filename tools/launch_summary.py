"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per-kernel totals / shares)."""
import csv, collections, sys
src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
h = None; agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0.0; n = 0
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows:
    if not r: continue
    if r[0] == "ID": h = r; continue
    if h is None: continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    name = d["Kernel Name"].split("(")[0][:58]
    agg[name][0] += 1; agg[name][1] += v; tot += v; n += 1
out = [f"# {src}: {n} launches, {tot:.1f} us total (ncu: cold-cache, serialised -> compare SHARES)"]
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k:58s} {c:5d} {t:11.1f} us {t / tot:6.1%}  avg {t / c:9.2f} us")
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out[:16]))
