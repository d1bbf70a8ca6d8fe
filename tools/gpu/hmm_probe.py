"""Can a kernel read the caller's pageable NumPy memory directly (HMM / ATS), and how fast?"""
import ctypes
import glob
import json
import os
import time

import numpy as np
import torch

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
    glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(cands[0])
torch.cuda.init()
out = {}
for name, attr in (("pageableMemoryAccess", 88), ("pageableMemoryAccessUsesHostPageTables", 100),
                   ("concurrentManagedAccess", 89), ("directManagedMemAccessFromHost", 101)):
    v = ctypes.c_int()
    rc = rt.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    out[name] = (rc, v.value)
n = (1 << 30) // 8
a = np.random.default_rng(0).standard_normal(n)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
# a torch "view" of host pageable memory as a CUDA tensor via __cuda_array_interface__
class CAI:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, True), "version": 3}
try:
    hv = torch.as_tensor(CAI(a.ctypes.data, n), device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(hv)  # device-side copy kernel reading host pageable memory
        torch.cuda.synchronize()
        out[f"kernel_read_pageable_GBps_{rep}"] = round(a.nbytes / (time.perf_counter() - t0) / 1e9, 2)
    out["correct"] = bool(torch.equal(dev.cpu(), torch.from_numpy(a)))
    # advise: keep the pages on the CPU, GPU accesses them remotely
    rc1 = rt.cudaMemAdvise(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 3, -1)  # SetPreferredLocation CPU
    rc2 = rt.cudaMemAdvise(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 5, 0)   # SetAccessedBy dev 0
    out["advise_rc"] = (rc1, rc2)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(hv)
        torch.cuda.synchronize()
        out[f"kernel_read_advised_GBps_{rep}"] = round(a.nbytes / (time.perf_counter() - t0) / 1e9, 2)
    t0 = time.perf_counter()
    s = float(a.sum())
    out["cpu_reread_GBps"] = round(a.nbytes / (time.perf_counter() - t0) / 1e9, 2)
except Exception as e:
    out["error"] = repr(e)[:300]
print(json.dumps(out))
