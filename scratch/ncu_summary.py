"""One-line key metrics per kernel from an ncu report (for profiles/ summaries)."""
import csv, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(h, row)); u = dict(zip(h, units))
        name = d.get("Kernel Name", "?").split("(")[0]
        parts = [f"{k}={d[k]}{(' ' + u[k]) if u.get(k) else ''}" for k in KEYS if k in d and d[k] != ""]
        print(f"{rep.split('/')[-1]} | {name} | " + "; ".join(parts))
