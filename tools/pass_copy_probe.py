"""Per-axis pass time vs a pure tile copy with the same access pattern (512^3).

    python tools/pass_copy_probe.py [--size 512] [--reps 20]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_04217_b200 import _dev, _lib  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dims = (a.size,) * 3
    n = a.size ** 3
    plan = _dev.plan_for(dims)
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    gb = 16.0 * n / 1e9
    ms = timed(lambda: y.copy_(x), a.reps)
    print(f"torch copy_ (contiguous)          {ms:.4f} ms  {gb / ms * 1e3:.0f} GB/s", flush=True)
    for axis in range(3):
        for mode, name in ((2, "tile copy"), (0, "synthesis"), (1, "analysis")):
            ms = timed(lambda: _lib.call("fl_axis_pass", plan.handle, axis, mode, _dev.ptr(x), _dev.ptr(y),
                                         _dev.stream()), a.reps)
            print(f"axis {axis} {name:10s}                 {ms:.4f} ms  {gb / ms * 1e3:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
