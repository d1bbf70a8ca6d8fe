"""Where the time of a small (latency-bound) solve goes: C1 1D 4096.

    python tools/c1_latency.py [--reps 20]

Prints one JSON line: the solve's median wall time, the per-IPM-iteration
wall times of the records, and the device time of the pieces an IPM
iteration launches (KKT matvec, the device-looped PCG of one Newton step,
the residual + assessment), each timed with CUDA events over many launches.
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import _lib, ipm, newton_system, workloads  # noqa: E402


def _events(fn, reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps  # us


def _wall(fn, reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e6 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--host-profile", action="store_true")
    a = ap.parse_args()
    inst = workloads.c1_1d(seed=0)
    mask = fl.Mask.from_bool(inst.flags, fl.GridShape(inst.dims))
    b = fl.observe(torch.from_numpy(inst.beta_true).cuda(), mask)
    b += torch.from_numpy(inst.noise).cuda()
    cfg = fl.IpmConfig(lam=inst.lam)
    out = {"config": "C1 1D 4096 lambda=0.3", "n": int(mask.shape.n)}
    for mode in (3, 2):
        _lib.call("fl_set_pcg_loop", mode)
        fl.solve(b, mask, cfg)
        ts, rep = [], None
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            _, rep = fl.solve(b, mask, cfg)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        key = "graph_loop" if mode == 3 else "host_loop"
        out[key] = {"solve_ms_median": statistics.median(ts) * 1e3, "solve_ms_min": min(ts) * 1e3,
                    "iterations": rep.iterations, "krylov": rep.krylov_counts,
                    "record_wall_us": [round(r.wall_time * 1e6, 1) for r in rep.records]}
    _lib.call("fl_set_pcg_loop", 3)
    n = mask.shape.n
    st = ipm.initial_state(b, mask, inst.lam)
    diag = newton_system.barrier_diagonals(st.s1, st.s2, st.nu1, st.nu2)
    db = torch.randn(n, dtype=torch.float64, device="cuda")
    dz = torch.randn(n, dtype=torch.float64, device="cuda")
    out["apply_kkt_us"] = {"device": _events(lambda: newton_system.apply_kkt(db, dz, diag, mask), 2000),
                           "wall": _wall(lambda: newton_system.apply_kkt(db, dz, diag, mask), 2000)}
    out["gram_us"] = {"device": _events(lambda: fl.gram(db, mask), 2000),
                      "wall": _wall(lambda: fl.gram(db, mask), 2000)}
    print(json.dumps(out), flush=True)




def host_profile(reps=50):
    """cProfile of `reps` C1 solves (host-side cost per IPM iteration)."""
    import cProfile
    import pstats

    inst = workloads.c1_1d(seed=0)
    mask = fl.Mask.from_bool(inst.flags, fl.GridShape(inst.dims))
    b = fl.observe(torch.from_numpy(inst.beta_true).cuda(), mask)
    b += torch.from_numpy(inst.noise).cuda()
    cfg = fl.IpmConfig(lam=inst.lam)
    fl.solve(b, mask, cfg)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(reps):
        fl.solve(b, mask, cfg)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(40)


if __name__ == "__main__":
    if "--host-profile" in sys.argv:
        host_profile()
    else:
        main()
