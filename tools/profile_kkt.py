"""Run a few KKT matvecs (or single passes) at side^3 for ncu / compute-sanitizer.

    python tools/profile_kkt.py [--size 512] [--reps 3] [--solve]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import _dev, _lib, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    side = args.size
    n = side ** 3
    shape = fl.GridShape((side,) * 3)
    mask = fl.Mask.from_bool(workloads.bragg_flags(side), shape)
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
    pkp = ctypes.c_double()
    for _ in range(args.reps):
        _lib.call("fl_kkt_apply", plan.handle, _dev.ptr(dm.bits), _dev.ptr(sig1), _dev.ptr(sig2),
                  _dev.ptr(d[:n]), _dev.ptr(d[n:]), _dev.ptr(top), _dev.ptr(bot), ctypes.byref(pkp),
                  _dev.stream())
    torch.cuda.synchronize()
    print(f"ok: {args.reps} KKT matvecs at {side}^3, d.Kd = {pkp.value:.6e}")


if __name__ == "__main__":
    main()
