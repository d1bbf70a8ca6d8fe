"""Time fl_residual_adjoint (A^T Z (b_hat - A beta)) and fl_gram at side^3 or --dims.

    python tools/time_resid.py [--size 512 | --dims 2048,2048] [--reps 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import _dev, _lib, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--dims", default=None, help="e.g. 2048,2048 (random 15%% mask)")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    if args.dims:
        import numpy as np

        dims = tuple(int(d) for d in args.dims.split(","))
        shape = fl.GridShape(dims)
        n = shape.n
        mask = fl.Mask.from_bool(np.random.default_rng(0).random(n) < 0.15, shape)
    else:
        side = args.size
        n = side ** 3
        shape = fl.GridShape((side,) * 3)
        mask = fl.Mask.from_bool(workloads.bragg_flags(side), shape)
    dm = mask.on_device()
    plan = _dev.plan_for(shape.dims)
    g = torch.Generator(device="cuda").manual_seed(0)
    bhat = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    beta = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    out = _dev.empty(n)
    s = _dev.stream()
    res = {}
    for name, fn in (("residual_adjoint", lambda: _lib.call("fl_residual_adjoint", plan.handle, _dev.ptr(dm.bits),
                                                            _dev.ptr(bhat), _dev.ptr(beta), _dev.ptr(out), s)),
                     ("gram", lambda: _lib.call("fl_gram", plan.handle, _dev.ptr(dm.bits), _dev.ptr(beta),
                                                _dev.ptr(out), s))):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / args.reps
    print({k: round(v, 4) for k, v in res.items()}, "ms")


if __name__ == "__main__":
    main()
