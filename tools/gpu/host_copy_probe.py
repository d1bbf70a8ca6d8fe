"""Host-side copy rates on the GPU box (what bounds the NumPy e2e of apply_kkt).

Pageable -> pinned memcpy with k threads, pinned H2D / D2H DMA alone and
concurrently, pageable H2D through the driver.  Prints one JSON line.
"""
import json
import os
import subprocess
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

GiB = 1 << 30
n = GiB // 8
src = np.random.default_rng(0).standard_normal(n)
dst = torch.empty(n, dtype=torch.float64, pin_memory=True)
dn = dst.numpy()
out = {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
try:
    out["lscpu"] = [l for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                    if any(k in l for k in ("Model name", "Socket", "NUMA node", "Thread(s)", "Core(s)"))]
except Exception:
    pass


def memcpy_rate(k, chunk=16 << 20):
    step = chunk // 8
    pieces = [(a, min(n, a + step)) for a in range(0, n, step)]
    with ThreadPoolExecutor(max_workers=k) as ex:
        for _ in range(2):
            t0 = time.perf_counter()
            list(ex.map(lambda p: np.copyto(dn[p[0]:p[1]], src[p[0]:p[1]]), pieces))
            dt = time.perf_counter() - t0
    return round(GiB / dt / 1e9, 1)


out["memcpy_GBps"] = {k: memcpy_rate(k) for k in (1, 2, 4, 8, 16, 24, 32, 48, 64) if k <= 2 * (os.cpu_count() or 1)}
dev = torch.empty(4 * n, dtype=torch.float64, device="cuda")
pin4 = torch.empty(4 * n, dtype=torch.float64, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


out["h2d_pinned_GBps"] = round(4 * GiB / timed(lambda: dev.copy_(pin4, non_blocking=True)) / 1e9, 1)
out["d2h_pinned_GBps"] = round(4 * GiB / timed(lambda: pin4.copy_(dev, non_blocking=True)) / 1e9, 1)


def both():
    with torch.cuda.stream(s1):
        dev[: 2 * n].copy_(pin4[: 2 * n], non_blocking=True)
    with torch.cuda.stream(s2):
        pin4[2 * n:].copy_(dev[2 * n:], non_blocking=True)


out["h2d_d2h_concurrent_GBps_each"] = round(2 * GiB / timed(both) / 1e9, 1)
src_t = torch.from_numpy(src)
out["h2d_pageable_driver_GBps"] = round(GiB / timed(lambda: dev[:n].copy_(src_t)) / 1e9, 1)
print(json.dumps(out))
