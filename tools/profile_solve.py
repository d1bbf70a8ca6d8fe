"""IPM solves of a BASELINE recipe (for an ncu launch list of the IPM/PCG kernels).

    python tools/profile_solve.py [--config c4] [--size 512] [--reps 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--host-pcg", action="store_true",
                    help="PCG host loop (fl_set_pcg_loop(2)) so a launch list sees every kernel launch")
    a = ap.parse_args()
    if a.host_pcg:
        from paper_2502_04217_b200 import _lib

        _lib.call("fl_set_pcg_loop", 2)
    inst = {"c1": lambda: workloads.c1_1d(seed=0), "c2": lambda: workloads.c2_2d(seed=0),
            "c3": lambda: workloads.c3_bragg(a.size, seed=0), "c4": lambda: workloads.c4_const(a.size)}[a.config]()
    mask = fl.Mask.from_bool(inst.flags, fl.GridShape(inst.dims))
    b = fl.observe(torch.from_numpy(inst.beta_true).cuda(), mask)
    b += torch.from_numpy(inst.noise).cuda()
    for _ in range(a.reps):
        beta, rep = fl.solve(b, mask, fl.IpmConfig(lam=inst.lam))
    torch.cuda.synchronize()
    print(f"ok: {rep.status} {rep.iterations} IPM, krylov {rep.krylov_counts}", flush=True)


if __name__ == "__main__":
    main()
