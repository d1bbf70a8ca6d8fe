"""One warm C4 solve at side^3 (for an ncu launch list of the IPM/PCG kernels).

    python tools/profile_solve.py [--size 512]
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
    a = ap.parse_args()
    inst = workloads.c4_const(a.size)
    mask = fl.Mask.from_bool(inst.flags, fl.GridShape(inst.dims))
    b = fl.observe(torch.from_numpy(inst.beta_true).cuda(), mask)
    b += torch.from_numpy(inst.noise).cuda()
    beta, rep = fl.solve(b, mask, fl.IpmConfig(lam=inst.lam))
    torch.cuda.synchronize()
    print(f"ok: {rep.status} {rep.iterations} IPM, krylov {rep.krylov_counts}", flush=True)


if __name__ == "__main__":
    main()
