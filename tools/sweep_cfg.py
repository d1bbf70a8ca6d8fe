"""Per-pass timing of the KKT matvec at 512^3 for every instantiated kernel
variant (FL_CFG_STRIDED / FL_CFG_CONTIG, see csrc/fl_fastpass.cu).

    python tools/sweep_cfg.py [--size 512] [--reps 10]
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
from paper_2502_04217_b200 import _dev, _lib, workloads  # noqa: E402

# cfg_code(t_sel, pipe, mb) = t_sel * 9 + pipe * 3 + mb - 1
VARIANTS = {10: "512thr/none/2", 5: "256thr/single/3", 7: "256thr/double/2", 12: "512thr/single/1",
            15: "512thr/double/1", 2: "256thr/none/3", 4: "256thr/single/2",
            28: "256thr/none/2/E16", 31: "256thr/single/2/E16", 36: "512thr/none/1/E16"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--reps", type=int, default=10)
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
    buf = (ctypes.c_double * 8)()
    cnt = ctypes.c_int()
    ref = None

    def run():
        acc = np.zeros(6)
        for i in range(args.reps + 2):
            _lib.call("fl_kkt_apply_profiled", plan.handle, _dev.ptr(dm.bits), _dev.ptr(sig1), _dev.ptr(sig2),
                      _dev.ptr(d[:n]), _dev.ptr(d[n:]), _dev.ptr(top), _dev.ptr(bot), buf, ctypes.byref(cnt),
                      _dev.stream())
            if i >= 2:
                acc += np.array(buf[:6])
        return acc / args.reps

    results = {}
    for which in ("FL_CFG_STRIDED", "FL_CFG_CONTIG"):
        for cfg, name in VARIANTS.items():
            os.environ[which] = str(cfg)
            ms = run()
            chk = top.clone()
            if ref is None:
                ref = chk
            err = float((chk - ref).abs().max())
            results[f"{which}={cfg} ({name})"] = [round(x, 4) for x in ms]
            print(f"{which}={cfg:2d} {name:18s} passes_ms={np.round(ms, 4).tolist()} total={ms.sum():.4f} "
                  f"maxdiff={err:.1e}", flush=True)
        del os.environ[which]
    for mm in ("0", "1", "2", "3", "4", "5", "6"):
        os.environ["FL_MIRROR"] = mm
        ms = run()
        err = float((top - ref).abs().max())
        results[f"FL_MIRROR={mm}"] = [round(x, 4) for x in ms]
        print(f"FL_MIRROR={mm} passes_ms={np.round(ms, 4).tolist()} total={ms.sum():.4f} maxdiff={err:.1e}",
              flush=True)
    del os.environ["FL_MIRROR"]
    print(json.dumps(results))


if __name__ == "__main__":
    main()
