"""Cost of page-locking a user NumPy array in place (cudaHostRegister) vs staging copies."""
import ctypes
import json
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so") if False else None
try:
    cudart = ctypes.CDLL("libcudart.so.12")
except OSError:
    import glob
    import os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    cands += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    cudart = ctypes.CDLL(cands[0])
torch.cuda.init()
out = {}
for gib in (1, 4):
    n = (gib << 30) // 8
    a = np.random.default_rng(0).standard_normal(n)
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        rc = cudart.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 0)
        t1 = time.perf_counter()
        dev.copy_(torch.from_numpy(a), non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rc2 = cudart.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
        t3 = time.perf_counter()
        out[f"{gib}GiB_rep{rep}"] = {"rc": rc, "register_GBps": round(a.nbytes / (t1 - t0) / 1e9, 1),
                                    "dma_GBps": round(a.nbytes / (t2 - t1) / 1e9, 1),
                                    "unregister_GBps": round(a.nbytes / (t3 - t2) / 1e9, 1), "rc2": rc2}
    # page-locked allocation of a fresh pinned buffer (torch host allocator, first use)
    t0 = time.perf_counter()
    p = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out[f"{gib}GiB_pin_alloc_GBps"] = round(a.nbytes / (time.perf_counter() - t0) / 1e9, 1)
    del p
print(json.dumps(out))
