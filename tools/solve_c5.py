"""C5 (1024^3 Bragg-punched, constant amplitudes, lambda = 0.5) IPM solve on ONE B200.

The solver's device footprint is 20 n doubles (160 B/voxel, ipm.Workspace +
b_hat): 172 GB at n = 1024^3, inside one 180 GB B200.  Inputs are the host
recipe (workloads.c4_const); the observation b = observe(beta_true) + noise is
formed on the GPU and brought back to the host so that nothing but the solver
holds device memory during the solve.

    python tools/solve_c5.py [--side 1024] [--out gpurun_out/solve_c5.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# 8 GiB vectors of several sizes come and go before the solve: let freed
# segments be remapped instead of fragmenting the 180 GB
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=1024)
    ap.add_argument("--out", default="gpurun_out/solve_c5.json")
    args = ap.parse_args()
    t0 = time.perf_counter()
    inst = workloads.c4_const(args.side)
    shape = fl.GridShape(inst.dims)
    mask = fl.Mask.from_bool(inst.flags, shape)
    del inst.flags
    t_gen = time.perf_counter() - t0
    bt = torch.from_numpy(inst.beta_true).cuda()
    b = fl.observe(bt, mask)
    del bt
    b += torch.from_numpy(inst.noise).cuda()
    b_host = b.cpu().numpy()
    del b
    torch.cuda.empty_cache()
    free0, total = torch.cuda.mem_get_info()
    torch.cuda.reset_peak_memory_stats()
    cfg = fl.IpmConfig(lam=inst.lam, tol=1e-8)
    times = []
    for _ in range(2):  # the first call also pins ~16 GB of host staging and builds plans/graphs
        beta = None
        t0 = time.perf_counter()
        beta, rep = fl.solve(b_host, mask, cfg)
        times.append(time.perf_counter() - t0)
        print(f"solve {len(times)}: {times[-1]:.2f} s, IPM loop {rep.wall_time:.2f} s, per iteration "
              f"{[round(r.wall_time, 3) for r in rep.records]}", flush=True)
    peak = torch.cuda.max_memory_allocated()
    true_support = np.flatnonzero(inst.beta_true)
    found = np.flatnonzero(np.abs(beta) > 1e-6 * np.max(np.abs(beta)))
    out = {
        "config": f"C5 recipe {args.side}^3 on one GPU, lambda={inst.lam}, tol=1e-8",
        "n": shape.n, "status": rep.status, "ipm_iterations": rep.iterations,
        "krylov": rep.krylov_counts, "total_krylov": rep.total_krylov,
        "solve_s_numpy_in_out": {"cold": round(times[0], 3), "warm": round(times[1], 3)},
        "host_generation_s": round(t_gen, 1),
        "final_objective": rep.final_objective,
        "support_exact": bool(np.array_equal(found, true_support)), "n_support": int(found.size),
        "device_peak_allocated_GB": round(peak / 1e9, 2), "device_total_GB": round(total / 1e9, 2),
        "device_free_before_GB": round(free0 / 1e9, 2),
    }
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
