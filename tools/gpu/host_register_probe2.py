"""Chunked cudaHostRegister/Unregister throughput with k threads, and a register -> DMA -> unregister pipeline."""
import ctypes
import glob
import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
    glob.glob("/usr/local/cuda/lib64/libcudart.so*")
cudart = ctypes.CDLL(cands[0])
torch.cuda.init()
PAGE = 4096
n = (4 << 30) // 8
a = np.random.default_rng(0).standard_normal(n)
base = a.ctypes.data
lo_al = (base + PAGE - 1) // PAGE * PAGE
hi_al = (base + a.nbytes) // PAGE * PAGE
out = {"base_mod_page": base % PAGE}


def chunks(mib):
    step = mib << 20
    return [(p, min(hi_al, p + step)) for p in range(lo_al, hi_al, step)]


def reg(c):
    return cudart.cudaHostRegister(ctypes.c_void_p(c[0]), ctypes.c_size_t(c[1] - c[0]), 0)


def unreg(c):
    return cudart.cudaHostUnregister(ctypes.c_void_p(c[0]))


for mib in (16, 64):
    for k in (1, 2, 4, 8):
        cs = chunks(mib)
        with ThreadPoolExecutor(k) as ex:
            t0 = time.perf_counter()
            rcs = list(ex.map(reg, cs))
            t1 = time.perf_counter()
            rcs2 = list(ex.map(unreg, cs))
            t2 = time.perf_counter()
        out[f"{mib}MiB_k{k}"] = {"reg_GBps": round((hi_al - lo_al) / (t1 - t0) / 1e9, 1),
                                 "unreg_GBps": round((hi_al - lo_al) / (t2 - t1) / 1e9, 1),
                                 "rc": max(rcs), "rc2": max(rcs2)}
# pipeline: workers register chunk i, main thread DMAs it as soon as it is registered,
# workers unregister after its copy event
dev = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
for mib, k in ((64, 4), (64, 8), (32, 8)):
    cs = chunks(mib)
    with ThreadPoolExecutor(k) as ex:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        futs = [ex.submit(reg, c) for c in cs]
        unf = []
        with torch.cuda.stream(s):
            for c, f in zip(cs, futs):
                f.result()
                i0, i1 = (c[0] - base) // 8, (c[1] - base) // 8
                dev[i0:i1].copy_(torch.from_numpy(a[i0:i1]), non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
                unf.append(ex.submit(lambda e=ev, cc=c: (e.synchronize(), unreg(cc))))
        for f in unf:
            f.result()
        torch.cuda.synchronize()
        out[f"pipeline_{mib}MiB_k{k}_GBps"] = round((hi_al - lo_al) / (time.perf_counter() - t0) / 1e9, 1)
print(json.dumps(out))
