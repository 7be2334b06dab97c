"""K1 steady-state: N back-to-back fused normal matvecs on the config-4 slice shape, each bracketed by CUDA
events; per-launch time distribution with nvidia-smi SM clock / power sampled during the run."""
import os
import subprocess
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14524_b200 import Context  # noqa: E402

m, n = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "50000x50000").split("x"))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 200
st = torch.cuda.Stream()
ctx = Context(0, stream=st)
lda = (m + 31) // 32 * 32
A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
d = torch.rand(n, dtype=torch.float64, device="cuda") + 0.1
v = torch.randn(m, dtype=torch.float64, device="cuda")
w = torch.empty(m, dtype=torch.float64, device="cuda")
byts = 8.0 * (m * n + n + 2 * m)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append(out)
        stop.wait(0.05)


torch.cuda.synchronize()
th = threading.Thread(target=sampler)
th.start()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
with torch.cuda.stream(st):
    ev[0].record(st)
    for i in range(N):
        ctx.nys_normal_matvec(A, lda, m, d, None, 1e-3, v, w)
        ev[i + 1].record(st)
torch.cuda.synchronize()
stop.set()
th.join()
t = np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(N)])
gbs = byts / (t * 1e-3) / 1e9
print(f"m={m} n={n}: per-launch ms: first5 {np.round(t[:5], 3).tolist()} | median {np.median(t):.3f} min {t.min():.3f} "
      f"max {t.max():.3f} | GB/s median {np.median(gbs):.0f} best {gbs.max():.0f} p10 {np.percentile(gbs, 10):.0f}")
if N >= 10:
    print("deciles of GB/s over the run:", [int(np.median(gbs[i * N // 10:(i + 1) * N // 10])) for i in range(10)])
print("smi samples (sm MHz, W, pcap):", samples[::max(1, len(samples) // 12)])
