"""NumPy-in/out apply_kkt at 512^3: staging slots x chunk size (upload_chunks tuning)."""
import json
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
res = {}
for slots, mib in [(8, 64), (16, 64), (16, 32), (32, 32), (32, 16), (12, 64), (24, 32)]:
    _dev._UPLOAD_SLOTS = slots
    _dev._STAGE_CHUNK = mib << 20
    for _ in range(2):
        t, b = apply_kkt(db, dz, diag, mask)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(6):
        t, b = apply_kkt(db, dz, diag, mask)
    torch.cuda.synchronize()
    res[f"{slots}x{mib}MiB"] = round(6 / (time.perf_counter() - t0), 2)
    print(json.dumps(res), flush=True)
