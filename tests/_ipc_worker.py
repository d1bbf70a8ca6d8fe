"""Worker of tests/test_gpu_sharded.py::test_peer_exchange_across_processes.

Two processes (torch.distributed.run, gloo group) share cuda:0: each owns one
slab rank of a ShardedGrid whose peer exchange runs over REAL CUDA-IPC
buffers -- every rank allocates its receive slabs, the handles are
all-gathered and opened in the other process (DistComm.peer_buffers), and the
transposing exchange kernels store straight into the other process's memory.
No kernel waits on another rank: the ranks meet only in host-side gloo
collectives after draining their streams (DistComm.barrier), so the two
processes may time-slice the GPU in any order.

Rank 0 prints one JSON line: the gathered sharded gram, residual pass, KKT
apply and sharded solve against the same computations with two emulated
ranks in one process (LocalComm(2): bitwise the same kernels) and against
the single-GPU package.
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import sharded as sh  # noqa: E402


def gather(t, world):
    h = t.cpu()
    out = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(out, h)
    return [o.numpy() for o in out]


def run(comm, dims, beta, flags, bfull, sig1, sig2, dz, P, lam, exchange="peer"):
    """Sharded gram, residual pass, KKT apply and solve on the ranks of ``comm``."""
    grid = sh.ShardedGrid(dims, comm, exchange=exchange)
    assert grid.exchange == exchange
    geo = grid.geo
    prob = sh.ShardedProblem.from_host(grid, flags, np.where(flags, 0.0, bfull))
    xb = [fl._dev.to_dev(geo.x_slab(beta, r)) for r in comm.ranks]
    g = [fl._dev.empty(geo.n_local) for _ in comm.ranks]
    nrm = grid.gram(xb, g, prob.bits_y, want_norm=True)
    res = {"gram": [t.clone() for t in g], "norm": nrm}
    grid.gram(xb, g, prob.bits_y, prob.bhat_y)
    res["resid"] = [t.clone() for t in g]
    s1 = [fl._dev.to_dev(geo.x_slab(sig1, r)) for r in comm.ranks]
    s2 = [fl._dev.to_dev(geo.x_slab(sig2, r)) for r in comm.ranks]
    zz = [fl._dev.to_dev(geo.x_slab(dz, r)) for r in comm.ranks]
    tops = [fl._dev.empty(geo.n_local) for _ in comm.ranks]
    bots = [fl._dev.empty(geo.n_local) for _ in comm.ranks]
    sh.kkt_apply(grid, prob.bits_y, s1, s2, xb, zz, tops, bots)
    res["top"], res["bottom"] = tops, bots
    betas, rep = sh.sharded_solve(prob, lam, fl.IpmConfig(lam=lam))
    res["beta"] = betas
    res["solve"] = (rep.status, rep.iterations, list(rep.krylov_counts), rep.final_objective)
    torch.cuda.synchronize()
    return geo, res


def main():
    dist.init_process_group("gloo")
    r, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dims = (32, 16, 24)
    rng = np.random.default_rng(11)  # the same draws on every rank
    n = int(np.prod(dims))
    beta = rng.standard_normal(n)
    flags = rng.random(n) < 0.15
    bfull = rng.standard_normal(n)
    sig1, sig2 = rng.random(n) + 0.5, rng.random(n) + 0.5
    dz = rng.standard_normal(n)
    lam = 0.5
    comm = sh.DistComm()  # host-side (gloo) group over GPU slabs
    geo, res = run(comm, dims, beta, flags, bfull, sig1, sig2, dz, world, lam)
    full = {k: geo.from_x(gather(res[k][0], world)) for k in ("gram", "resid", "top", "bottom", "beta")}
    comm.release_peer_buffers()
    # the NCCL-free fallback exchange (pack -> all-to-all -> unpack) across the processes
    geo2, res2 = run(comm, dims, beta, flags, bfull, sig1, sig2, dz, world, lam, exchange="a2a")
    full2 = {k: geo2.from_x(gather(res2[k][0], world)) for k in ("gram", "resid", "top", "bottom", "beta")}
    # the drop-in API across the processes: root holds the reference arguments
    mask_full = fl.Mask.from_bool(flags, fl.GridShape(dims))
    b_obs = bfull[~flags]
    beta_d, rep_d = sh.solve(b_obs if r == 0 else None, mask_full if r == 0 else None, fl.IpmConfig(lam=lam),
                             comm=sh.DistComm())
    if r == 0:
        beta_1, rep_1 = fl.solve(b_obs, mask_full, fl.IpmConfig(lam=lam))
        dropin = {"status": [rep_d.status, rep_1.status], "iterations": [rep_d.iterations, rep_1.iterations],
                  "krylov": [list(rep_d.krylov_counts), list(rep_1.krylov_counts)],
                  "objective_rel": abs(rep_d.final_objective - rep_1.final_objective) / abs(rep_1.final_objective),
                  "beta_rel_l2": float(np.linalg.norm(beta_d - beta_1) / np.linalg.norm(beta_1))}
        _, emu = run(sh.LocalComm(world), dims, beta, flags, bfull, sig1, sig2, dz, world, lam)
        efull = {k: geo.from_x([t.cpu().numpy() for t in emu[k]]) for k in full}
        mask = fl.Mask.from_bool(flags, fl.GridShape(dims))
        single = np.asarray(fl.gram(beta, mask))
        out = {"world": world,
               "bitwise_vs_emulated": {k: bool(np.array_equal(full[k], efull[k])) for k in full},
               "a2a_bitwise_vs_peer": {k: bool(np.array_equal(full2[k], full[k])) for k in full},
               "norm_equal": res["norm"] == emu["norm"],
               "solve": res["solve"], "solve_emulated": emu["solve"],
               "gram_vs_single_gpu": float(np.max(np.abs(full["gram"] - single)) / np.abs(single).max()),
               "dropin_vs_single_gpu": dropin}
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
