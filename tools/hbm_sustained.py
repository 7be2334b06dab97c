"""HBM bandwidth burst vs sustained on this box: torch copy of 1 Gi bf16 elements (read + write bytes, the
MEASURED_PEAKS.json recipe) and a read-only sum of 4 GB, each timed per launch back to back for ~4 s with
CUDA events; nvidia-smi SM clock / power sampled meanwhile."""
import subprocess
import threading
import time

import numpy as np
import torch

samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append(subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                                       "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip())
        stop.wait(0.1)


a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda").normal_()
b = torch.empty_like(a)
big = torch.ones(1 << 29, dtype=torch.float64, device="cuda")
out = torch.empty((), dtype=torch.float64, device="cuda")
for name, fn, byts in [("copy", lambda: b.copy_(a), 2 * a.numel() * 2), ("read_sum", lambda: torch.sum(big, dim=0, out=out), big.numel() * 8)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    time.sleep(2.0)            # let the clocks settle back (idle)
    th = threading.Thread(target=sampler)
    samples.clear(); stop.clear(); th.start()
    ts = []
    t0 = time.time()
    while time.time() - t0 < 4.0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    stop.set(); th.join()
    g = byts / np.array(ts) / 1e9
    print(f"{name}: burst (best of first 10) {g[:10].max():.0f} GB/s | sustained median {np.median(g):.0f} | last-second median "
          f"{np.median(g[-len(g) // 4:]):.0f} | n={len(g)} | clocks {samples[::max(1, len(samples) // 8)]}", flush=True)
