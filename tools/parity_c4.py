"""C4 trajectory parity at full size: B200 solve vs the CPU oracle, K IPM iterations.

SURVEY §8(d) "C4 fallback": the full 512^3 CPU solve does not fit a test
budget, so both sides run the C4 recipe (512^3 Bragg-punched, constant
amplitudes, lambda = 0.5) for ``--iters`` IPM iterations (max_iters = K; the
best iterate is returned on both sides) and every per-iteration record is
compared.  Needs ~100 GB of host RAM for the oracle (the GPU box has it).

    python tools/parity_c4.py [--side 512] [--iters 3] [--out gpurun_out/parity_c4_512.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from oracle import fftlasso_oracle as orc  # noqa: E402
from paper_2502_04217_b200 import workloads  # noqa: E402

KEYS = ("mu", "primal_inf", "dual_inf", "complementarity", "kkt_max", "alpha_primal", "alpha_dual",
        "pcg_residual")


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=512)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/parity_c4_512.json")
    args = ap.parse_args()
    inst = workloads.c4_const(args.side)
    dims = inst.dims
    om = orc.make_mask(dims, flags=inst.flags)
    b = orc.observe(inst.beta_true, om) + inst.noise

    t0 = time.perf_counter()
    beta_g, rep_g = fl.solve(b, fl.Mask.from_bool(inst.flags, fl.GridShape(dims)),
                             fl.IpmConfig(lam=inst.lam, tol=1e-8, max_iters=args.iters))
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    beta_c, rep_c = orc.solve(b, om, orc.OConfig(lam=inst.lam, tol=1e-8, max_iters=args.iters))
    t_cpu = time.perf_counter() - t0

    rows = []
    for rg, rc in zip(rep_g.records, rep_c.records):
        rg = rg.to_dict()
        rows.append({"iteration": rc["iteration"], "krylov_gpu": rg["krylov_iters"],
                     "krylov_cpu": rc["krylov_iters"],
                     **{f"rel_{k}": rel(rg[k], rc[k]) for k in KEYS}})
    sup_g = orc.support(beta_g)[:2]
    sup_c = orc.support(beta_c)[:2]
    out = {
        "config": f"C4 recipe {args.side}^3, lambda={inst.lam}, tol=1e-8, max_iters={args.iters}",
        "status": [rep_g.status, rep_c.status],
        "iterations": [rep_g.iterations, rep_c.iterations],
        "krylov_equal": rep_g.krylov_counts == rep_c.krylov_counts,
        "krylov_gpu": rep_g.krylov_counts, "krylov_cpu": rep_c.krylov_counts,
        "objective_rel_diff": rel(rep_g.final_objective, rep_c.final_objective),
        "beta_rel_l2": float(np.linalg.norm(beta_g - beta_c) / np.linalg.norm(beta_c)),
        "support_equal": bool(all(np.array_equal(a, c) for a, c in zip(sup_g, sup_c))),
        "n_support": int(sum(a.size for a in sup_c)),
        "per_iteration": rows,
        "seconds": {"gpu_solve": round(t_gpu, 3), "cpu_oracle_solve": round(t_cpu, 1)},
    }
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
