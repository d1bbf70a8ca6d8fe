"""Per-pass CUDA-event times of the KKT matvec at side^3 (fl_kkt_apply_profiled).

    python tools/pass_times.py [--size 512] [--reps 10]

Prints one JSON line: per-pass ms, GB/s against the algorithmic bytes
(16 B/voxel per transform pass, +n/8 mask bytes for the fused pass, 56 B/voxel
for the epilogue) and the matvec total.
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import _dev, _lib  # noqa: E402

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    side = args.size
    n = side ** 3
    shape = fl.GridShape((side,) * 3)
    from paper_2502_04217_b200.masking import BraggMask

    mask = BraggMask(shape)
    dm = mask.on_device()
    plan = _dev.plan_for(shape.dims)
    gen = torch.Generator(device="cuda").manual_seed(0)
    s = [torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) + 0.4 for _ in range(4)]
    sig1, sig2 = _dev.empty(n), _dev.empty(n)
    _lib.call("fl_barrier_diagonals", n, *(_dev.ptr(t) for t in s), _dev.ptr(sig1), _dev.ptr(sig2),
              None, None, None, None, _dev.stream())
    del s
    d = torch.randn(2 * n, dtype=torch.float64, device="cuda", generator=gen)
    top, bot = _dev.empty(n), _dev.empty(n)
    buf = (ctypes.c_double * 8)()
    cnt = ctypes.c_int()
    from bench import pass_layout

    names, alg = pass_layout(plan.handle, n, 3)
    acc = np.zeros(len(names))
    for i in range(args.reps + 3):
        _lib.call("fl_kkt_apply_profiled", plan.handle, _dev.ptr(dm.bits), _dev.ptr(sig1), _dev.ptr(sig2),
                  _dev.ptr(d[:n]), _dev.ptr(d[n:]), _dev.ptr(top), _dev.ptr(bot), buf, ctypes.byref(cnt),
                  _dev.stream())
        if i >= 3:
            acc += np.array(buf[:len(names)])
    ms = acc / args.reps
    out = {"size": side, "order": "B" if names[-1].endswith("kkt_epilogue") and len(names) == 5 else "A",
           "passes": {k: {"ms": round(float(m), 4), "GBps": round(a / m / 1e6, 1)}
                      for k, m, a in zip(names, ms, alg)},
           "total_ms": round(float(ms.sum()), 4), "matvec_per_s": round(1e3 / float(ms.sum()), 2)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
