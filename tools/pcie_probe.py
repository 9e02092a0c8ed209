"""Host<->device copy bandwidth on the box: pinned vs pageable, plus host
memcpy (the staging cost of a pageable end-to-end call)."""
import os, subprocess, time
import numpy as np
import torch

def bw(fn, nbytes, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return nbytes / best / 1e9

n = 1 << 26
d = torch.empty(n, dtype=torch.float64, device="cuda")
hp = torch.empty(n, dtype=torch.float64).pin_memory()
hn = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n))
out = {}
out["h2d_pinned"] = bw(lambda: d.copy_(hp, non_blocking=True), 8 * n)
out["d2h_pinned"] = bw(lambda: hp.copy_(d, non_blocking=True), 8 * n)
out["h2d_pageable"] = bw(lambda: d.copy_(hn), 8 * n)
out["d2h_pageable"] = bw(lambda: hn.copy_(d), 8 * n)
a = np.random.default_rng(2).uniform(-1, 1, n); b = np.empty_like(a)
t0 = time.perf_counter(); np.copyto(b, a); out["host_memcpy_1t_warm"] = 8 * n / (time.perf_counter() - t0) / 1e9
c = np.empty_like(a)
t0 = time.perf_counter(); np.copyto(c, a); out["host_memcpy_1t_cold_dst"] = 8 * n / (time.perf_counter() - t0) / 1e9
from concurrent.futures import ThreadPoolExecutor
T = os.cpu_count()
pool = ThreadPoolExecutor(T)
sp = np.linspace(0, n, T + 1).astype(int)
def par():
    list(pool.map(lambda i: np.copyto(b[sp[i]:sp[i+1]], a[sp[i]:sp[i+1]]), range(T)))
par(); t0 = time.perf_counter(); par(); out[f"host_memcpy_{T}t"] = 8 * n / (time.perf_counter() - t0) / 1e9
for k, v in out.items():
    print(f"{k:28s} {v:8.2f} GB/s")
print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout)
print(subprocess.run(["nproc"], capture_output=True, text=True).stdout)
print(subprocess.run(["bash", "-c", "lscpu | head -20; nvidia-smi topo -m; cat /proc/meminfo | head -3"], capture_output=True, text=True).stdout)
