"""Per-axis-pass parity vs the oracle on shapes with many tiles per CTA."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from oracle import fftlasso_oracle as orc  # noqa: E402
from paper_2502_04217_b200 import _dev, _lib  # noqa: E402

rng = np.random.default_rng(0)
for cfgs in [None, ("FL_CFG_CONTIG", "5"), ("FL_CFG_CONTIG", "10"), ("FL_CFG_STRIDED", "15")]:
    if cfgs:
        os.environ[cfgs[0]] = cfgs[1]
    for dims in [(512, 64, 64), (256, 256, 64), (1024, 64, 16), (64, 64, 512)]:
        shape = fl.GridShape(dims)
        plan = _dev.plan_for(dims)
        b = rng.standard_normal(shape.n)
        grid = b.reshape(dims)
        for ax in range(3):
            for an in (0, 1):
                src = torch.from_numpy(b).cuda()
                dst = torch.empty_like(src)
                _lib.call("fl_axis_pass", plan.handle, ax, an, _dev.ptr(src), _dev.ptr(dst), _dev.stream())
                ref = (orc.analyze_axis if an else orc.synth_axis)(grid, ax).reshape(-1)
                err = float(np.max(np.abs(dst.cpu().numpy() - ref)))
                if err > 1e-12:
                    bad = np.flatnonzero(np.abs(dst.cpu().numpy() - ref) > 1e-9)
                    print(cfgs, dims, "axis", ax, "analysis" if an else "synth", f"err {err:.2e}",
                          "first bad", bad[:4], "count", bad.size, flush=True)
    if cfgs:
        del os.environ[cfgs[0]]
print("done")
