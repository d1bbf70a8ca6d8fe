"""Worker for tests/test_sharded_gloo.py (launched by torch.distributed.run)."""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from helpers.numpy_shard_ops import NumpyShardOps, ShmPeerComm  # noqa: E402
from oracle import fftlasso_oracle as orc  # noqa: E402
from paper_2502_04217_b200.sharded import MAX, MIN, SUM, DistComm, ShardedGrid, ShardedProblem  # noqa: E402


def main():
    dist.init_process_group("gloo")
    r = dist.get_rank()
    out = {}
    raw = {}
    for dims, exchange in [(d, ex) for d in [(4, 6, 8), (8, 4, 6), (16, 16, 8)] for ex in ("a2a", "peer")]:
        comm = DistComm() if exchange == "a2a" else ShmPeerComm()
        grid = ShardedGrid(dims, comm, ops_factory=NumpyShardOps, exchange=exchange)
        geo = grid.geo
        rng = np.random.default_rng(7)  # same on every rank
        n = geo.n
        beta = rng.standard_normal(n)
        flags = rng.random(n) < 0.2
        bfull = rng.standard_normal(n)
        om = orc.make_mask(dims, flags=flags)
        bhat = np.where(flags, 0.0, bfull)
        prob = ShardedProblem.from_host(grid, flags, bhat)
        xb = [NumpyShardOps.vec(geo.x_slab(beta, rk)) for rk in comm.ranks]
        g = [NumpyShardOps.empty(geo.n_local) for _ in comm.ranks]
        nrm = grid.gram(xb, g, prob.bits_y, want_norm=True)
        ref = orc.gram(beta, om)
        err_gram = float(np.max(np.abs(g[0].numpy() - geo.x_slab(ref, r))))
        ax = orc.synthesize(beta, dims)
        err_nrm = abs(nrm - float(np.sum(ax[~flags] ** 2))) / max(1.0, nrm)
        gr = [NumpyShardOps.empty(geo.n_local) for _ in comm.ranks]
        grid.gram(xb, gr, prob.bits_y, prob.bhat_y)
        ref_r = orc.observe_adjoint(bfull[~flags] - orc.observe(beta, om), om)
        err_resid = float(np.max(np.abs(gr[0].numpy() - geo.x_slab(ref_r, r))))
        y = [NumpyShardOps.empty(geo.n_local) for _ in comm.ranks]
        grid.synthesize_to_y(xb, y)
        err_syn = float(np.max(np.abs(y[0].numpy() - geo.y_slab(ax, r))))
        red = [comm.reduce([[float(r + 1)]], op)[0] for op in (SUM, MAX, MIN)]
        import torch

        td = torch.tensor([float(r + 1), 0.5 * (r + 1)], dtype=torch.float64)
        comm.reduce_device([td])  # the device-scalar PCG's all-reduce (gloo: CPU tensors)
        red += td.tolist()
        out[f"{dims} {exchange}"] = dict(gram=err_gram, norm=err_nrm, resid=err_resid, synth=err_syn, red=red)
        raw[(dims, exchange)] = (g[0].numpy().tobytes(), gr[0].numpy().tobytes(), y[0].numpy().tobytes(), nrm)
        if exchange == "peer":
            out[f"{dims} peer==a2a"] = raw[(dims, "peer")] == raw[(dims, "a2a")]
            comm.close()
    if r == 0:
        print("RESULT " + json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
