"""NumPy-in/out apply_kkt at 512^3 with different staging thread counts (e2e probe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import _dev  # noqa: E402
from paper_2502_04217_b200.masking import BraggMask  # noqa: E402
from paper_2502_04217_b200.newton_system import BarrierDiagonals, apply_kkt  # noqa: E402

n = 512 ** 3
mask = BraggMask(fl.GridShape((512,) * 3))
rng = np.random.default_rng(0)
db, dz = rng.standard_normal(n), rng.standard_normal(n)
s1, s2 = rng.random(n) + 0.4, rng.random(n) + 0.4
diag = BarrierDiagonals(s1, s2, None, None, None, None)
for workers in (4, 8, 12, 16):
    _dev._POOL_WORKERS = workers
    _dev._pool = None
    for _ in range(2):
        apply_kkt(db, dz, diag, mask)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        t, b = apply_kkt(db, dz, diag, mask)
    torch.cuda.synchronize()
    print(f"workers {workers}: {5 / (time.perf_counter() - t0):.2f} matvec/s", flush=True)
