"""Probe: do two strided passes on an L2-sized column chunk cost ~one HBM pass?

Times synth axis 0 + synth axis 1 (in place) over 16 separate 512x512x32
arrays (64 MB each, 1 GiB total) against the same two passes on one 512^3
array.  If the chunk's intermediate stays in the 126 MB L2, the chunked
pair should cost about one HBM round trip instead of two.

    python tools/l2_chunk_probe.py [--k 32] [--reps 5]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_04217_b200 import _dev, _lib  # noqa: E402


def plan(dims):
    arr = (ctypes.c_int64 * 3)(*dims)
    h = ctypes.c_void_p()
    _lib.call("fl_plan_create", 3, arr, torch.cuda.current_device(), ctypes.byref(h))
    return h


def timed(fn, reps):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    s = _dev.stream()
    full = torch.randn(512 ** 3, dtype=torch.float64, device="cuda")
    pf = plan((512, 512, 512))
    nchunk = 512 // a.k
    chunks = [torch.randn(512 * 512 * a.k, dtype=torch.float64, device="cuda") for _ in range(nchunk)]
    pc = plan((512, 512, a.k))

    def two_full():
        _lib.call("fl_axis_pass", pf, 0, 0, _dev.ptr(full), _dev.ptr(full), s)
        _lib.call("fl_axis_pass", pf, 1, 0, _dev.ptr(full), _dev.ptr(full), s)

    def two_chunked():
        for c in chunks:
            _lib.call("fl_axis_pass", pc, 0, 0, _dev.ptr(c), _dev.ptr(c), s)
            _lib.call("fl_axis_pass", pc, 1, 0, _dev.ptr(c), _dev.ptr(c), s)

    def one_full():
        _lib.call("fl_axis_pass", pf, 0, 0, _dev.ptr(full), _dev.ptr(full), s)

    def one_chunked():
        for c in chunks:
            _lib.call("fl_axis_pass", pc, 0, 0, _dev.ptr(c), _dev.ptr(c), s)

    r = {"full: axis0+axis1": timed(two_full, a.reps), "full: axis0": timed(one_full, a.reps),
         f"chunked k={a.k}: axis0+axis1": timed(two_chunked, a.reps),
         f"chunked k={a.k}: axis0": timed(one_chunked, a.reps)}
    for k, v in r.items():
        print(f"{k:32s} {v:.4f} ms")


if __name__ == "__main__":
    main()
