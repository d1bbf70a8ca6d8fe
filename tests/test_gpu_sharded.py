"""GPU: slab-sharded operators and solve with P emulated ranks on one GPU.

LocalComm keeps all P shards in one process (no kernel waits on another
rank), so the CUDA slab transposes, the X-slab passes and the Y-slab fused
pass are checked against the oracle on the full grid, and the sharded IPM
solve against the single-GPU solve.
"""

import json

import numpy as np
import pytest

from conftest import load_golden
from oracle import fftlasso_oracle as orc

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_2502_04217_b200")
from paper_2502_04217_b200 import sharded as sh  # noqa: E402


@pytest.mark.parametrize("exchange", ["a2a", "peer"])
@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("dims", [(8, 8, 16), (16, 32, 64), (64, 64, 64), (128, 32, 512), (96, 40, 24)])
def test_sharded_operators_match_oracle(P, dims, exchange):
    if dims[0] % P or dims[1] % P:
        pytest.skip("not divisible")
    comm = sh.LocalComm(P)
    grid = sh.ShardedGrid(dims, comm, exchange=exchange)
    geo = grid.geo
    rng = np.random.default_rng(P * 1000 + dims[2])
    beta = rng.standard_normal(geo.n)
    flags = rng.random(geo.n) < 0.15
    bfull = rng.standard_normal(geo.n)
    om = orc.make_mask(dims, flags=flags)
    prob = sh.ShardedProblem.from_host(grid, flags, np.where(flags, 0.0, bfull))
    xb = [fl._dev.to_dev(geo.x_slab(beta, r)) for r in comm.ranks]
    g = [fl._dev.empty(geo.n_local) for _ in comm.ranks]
    nrm = grid.gram(xb, g, prob.bits_y, want_norm=True)
    ref = orc.gram(beta, om)
    got = geo.from_x([t.cpu().numpy() for t in g])
    tol = 1e-12 * np.abs(beta).max()
    assert np.max(np.abs(got - ref)) <= tol
    ax = orc.synthesize(beta, dims)
    assert abs(nrm - np.sum(ax[~flags] ** 2)) <= 1e-12 * nrm
    grid.gram(xb, g, prob.bits_y, prob.bhat_y)
    ref_r = orc.observe_adjoint(bfull[~flags] - orc.observe(beta, om), om)
    assert np.max(np.abs(geo.from_x([t.cpu().numpy() for t in g]) - ref_r)) <= 1e-12 * np.abs(ref_r).max()
    ys = [fl._dev.empty(geo.n_local) for _ in comm.ranks]
    grid.synthesize_to_y(xb, ys)
    for r in comm.ranks:
        assert np.max(np.abs(ys[r].cpu().numpy() - geo.y_slab(ax, r))) <= tol


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_solve_matches_single_gpu(P):
    g = load_golden("solve_c4_32")
    dims = tuple(int(d) for d in g["dims"])
    mask = fl.Mask(g["missing"], fl.GridShape(dims))
    lam = float(g["lam"])
    beta1, rep1 = fl.solve(g["b"], mask, fl.IpmConfig(lam=lam))
    comm = sh.LocalComm(P)
    grid = sh.ShardedGrid(dims, comm)
    bhat = np.zeros(mask.shape.n)
    bhat[~mask.missing_bool] = g["b"]
    prob = sh.ShardedProblem.from_host(grid, mask.missing_bool, bhat)
    betas, rep = sh.sharded_solve(prob, lam, fl.IpmConfig(lam=lam))
    beta = grid.geo.from_x([t.cpu().numpy() for t in betas])
    assert rep.status == rep1.status == "converged"
    assert rep.iterations == rep1.iterations
    assert all(abs(a - b) <= 1 for a, b in zip(rep.krylov_counts, rep1.krylov_counts))
    assert abs(rep.final_objective - rep1.final_objective) <= 1e-9 * abs(rep1.final_objective)
    assert np.linalg.norm(beta - beta1) <= 1e-8 * np.linalg.norm(beta1)
    ref = [r["krylov_iters"] for r in json.loads(str(g["records_json"]))]
    assert abs(rep.iterations - len(ref)) <= 1


@pytest.mark.parametrize("P", [2, 4, 8])
def test_peer_exchange_bitwise_equals_all_to_all(P):
    """The fused peer-store exchange (one transposing kernel per direction)
    gives exactly the pack / all-to-all / unpack results: gram, residual
    pass and synthesis to Y, at a grid whose 32-wide tiles straddle ranks."""
    dims = (8 * P * 3, 8 * P, 48)
    rng = np.random.default_rng(P)
    out = {}
    for ex in ("a2a", "peer"):
        comm = sh.LocalComm(P)
        grid = sh.ShardedGrid(dims, comm, exchange=ex)
        geo = grid.geo
        beta = np.random.default_rng(1).standard_normal(geo.n)
        flags = np.random.default_rng(2).random(geo.n) < 0.15
        bfull = np.random.default_rng(3).standard_normal(geo.n)
        prob = sh.ShardedProblem.from_host(grid, flags, np.where(flags, 0.0, bfull))
        xb = [fl._dev.to_dev(geo.x_slab(beta, r)) for r in comm.ranks]
        g = [fl._dev.empty(geo.n_local) for _ in comm.ranks]
        nrm = grid.gram(xb, g, prob.bits_y, want_norm=True)
        a = geo.from_x([t.cpu().numpy() for t in g])
        grid.gram(xb, g, prob.bits_y, prob.bhat_y)
        b = geo.from_x([t.cpu().numpy() for t in g])
        ys = [fl._dev.empty(geo.n_local) for _ in comm.ranks]
        grid.synthesize_to_y(xb, ys)
        out[ex] = (nrm, a.tobytes(), b.tobytes(), b"".join(y.cpu().numpy().tobytes() for y in ys))
    del rng
    assert out["a2a"] == out["peer"]


def test_sharded_solve_peer_exchange_equals_a2a():
    g = load_golden("solve_c4_32")
    dims = tuple(int(d) for d in g["dims"])
    mask = fl.Mask(g["missing"], fl.GridShape(dims))
    lam = float(g["lam"])
    bhat = np.zeros(mask.shape.n)
    bhat[~mask.missing_bool] = g["b"]
    res = {}
    for ex in ("a2a", "peer"):
        grid = sh.ShardedGrid(dims, sh.LocalComm(4), exchange=ex)
        prob = sh.ShardedProblem.from_host(grid, mask.missing_bool, bhat)
        betas, rep = sh.sharded_solve(prob, lam, fl.IpmConfig(lam=lam))
        res[ex] = (rep.krylov_counts, rep.final_objective, b"".join(t.cpu().numpy().tobytes() for t in betas))
    assert res["a2a"] == res["peer"]


def test_overlapped_forward_exchange_bitwise():
    """synth_x + X->Y exchange in plane chunks on two streams == one shot."""
    dims = (64, 32, 48)
    out = {}
    for k in (1, 4):
        comm = sh.LocalComm(2)
        grid = sh.ShardedGrid(dims, comm, exchange="peer", chunks=k)
        geo = grid.geo
        beta = np.random.default_rng(5).standard_normal(geo.n)
        flags = np.random.default_rng(6).random(geo.n) < 0.15
        prob = sh.ShardedProblem.from_host(grid, flags, np.where(flags, 0.0, 1.0))
        xb = [fl._dev.to_dev(geo.x_slab(beta, r)) for r in comm.ranks]
        g = [fl._dev.empty(geo.n_local) for _ in comm.ranks]
        nrm = grid.gram(xb, g, prob.bits_y, want_norm=True)
        out[k] = (nrm, b"".join(t.cpu().numpy().tobytes() for t in g))
    assert out[1] == out[4]


def test_sharded_solve_8_ranks_c4_recipe_64():
    """The C5 configuration's rank count (P = 8, peer exchange, chunked
    forward overlap forced on) on the C4 recipe at 64^3 against the
    single-GPU solve."""

    from paper_2502_04217_b200 import workloads

    inst = workloads.c4_const(64)
    shape = fl.GridShape(inst.dims)
    mask = fl.Mask.from_bool(inst.flags, shape)
    b = fl.observe(inst.beta_true, mask) + inst.noise
    beta1, rep1 = fl.solve(b, mask, fl.IpmConfig(lam=inst.lam))
    grid = sh.ShardedGrid(inst.dims, sh.LocalComm(8), exchange="peer", chunks=2)
    bhat = np.zeros(shape.n)
    bhat[~inst.flags] = b
    prob = sh.ShardedProblem.from_host(grid, inst.flags, bhat)
    betas, rep = sh.sharded_solve(prob, inst.lam, fl.IpmConfig(lam=inst.lam))
    beta = grid.geo.from_x([t.cpu().numpy() for t in betas])
    assert rep.status == rep1.status == "converged" and rep.iterations == rep1.iterations
    assert all(abs(x - y) <= 1 for x, y in zip(rep.krylov_counts, rep1.krylov_counts))
    assert abs(rep.final_objective - rep1.final_objective) <= 1e-9 * abs(rep1.final_objective)
    assert np.linalg.norm(beta - beta1) <= 1e-8 * np.linalg.norm(beta1)


def test_noise_is_a_function_of_the_global_voxel():
    """fl_noisy_embed: full grid vs X-slabs vs Y-slabs give bitwise the same
    noisy, masked volume (the draws are keyed by the global voxel index)."""
    import torch

    from paper_2502_04217_b200 import workloads

    dims = (32, 64, 48)
    d0, d1, d2 = dims
    P = 4
    geo = sh.SlabGeometry(dims, P)
    flags = np.random.default_rng(9).random(geo.n) < 0.2
    x = np.random.default_rng(10).standard_normal(geo.n)
    full = fl._dev.to_dev(x)
    bits = torch.from_numpy(sh.pack_bits(flags)).cuda()
    workloads.noisy_embed_device(full, bits, dims, (0, 0, 0), (d1 * d2, d2, 1), 77)
    ref = full.cpu().numpy()
    assert np.all(ref[flags] == 0.0)
    noise = (ref - x)[~flags]
    assert abs(noise.std() / 0.05 - 1) < 0.05 and abs(noise.mean()) < 0.01 * 0.05 * 10
    for r in range(P):
        xs = fl._dev.to_dev(geo.x_slab(x, r).copy())
        bx = torch.from_numpy(sh.pack_bits(geo.x_slab(flags, r))).cuda()
        workloads.noisy_embed_device(xs, bx, (geo.a, d1, d2), (r * geo.a, 0, 0), (d1 * d2, d2, 1), 77)
        assert xs.cpu().numpy().tobytes() == geo.x_slab(ref, r).tobytes()
        ys = fl._dev.to_dev(geo.y_slab(x, r))
        by = torch.from_numpy(sh.pack_bits(geo.y_slab(flags.astype(np.uint8), r))).cuda()
        workloads.noisy_embed_device(ys, by, (geo.b, d2, d0), (r * geo.b, 0, 0), (d2, 1, d1 * d2), 77)
        assert ys.cpu().numpy().tobytes() == geo.y_slab(ref, r).tobytes()


def test_sharded_solve_8_ranks_device_inputs_256():
    """The C5 pipeline at 256^3 with P = 8 emulated ranks (LocalComm, peer
    exchange): inputs generated on the device straight into slab layout
    (sharded.c4_problem_device) against the single-GPU device recipe
    (workloads.c4_const_device) -- same mask bits and b_hat, same solve."""
    import torch

    from paper_2502_04217_b200 import workloads

    side = 256
    mask, b, idx, _, lam = workloads.c4_const_device(side)
    beta1, rep1 = fl.solve(b, mask, fl.IpmConfig(lam=lam))
    dm = mask.on_device()
    bhat = torch.zeros(side ** 3, dtype=torch.float64, device="cuda")
    fl._lib.call("fl_embed", side ** 3, fl._dev.ptr(dm.bits), fl._dev.ptr(dm.offsets), fl._dev.ptr(b),
                 fl._dev.ptr(bhat), fl._dev.stream())
    bhat = bhat.cpu().numpy()
    flags = mask.missing_bool
    del b, dm
    grid = sh.ShardedGrid((side,) * 3, sh.LocalComm(8), exchange="peer")
    prob, idx2, _, lam2 = sh.c4_problem_device(grid, noise_seed=0)
    assert lam2 == lam and np.array_equal(idx, idx2)
    geo = grid.geo
    for r in range(8):
        want = sh.pack_bits(geo.y_slab(flags.astype(np.uint8), r))
        assert prob.bits_y[r].cpu().numpy().tobytes() == want.tobytes()
        got = prob.bhat_y[r].cpu().numpy()
        exp = geo.y_slab(bhat, r)
        assert np.max(np.abs(got - exp)) <= 1e-12 * np.abs(exp).max()
    betas, rep = sh.sharded_solve(prob, lam, fl.IpmConfig(lam=lam))
    assert rep.status == rep1.status == "converged"
    assert abs(rep.iterations - rep1.iterations) <= 1
    assert all(abs(x - y) <= 1 for x, y in zip(rep.krylov_counts, rep1.krylov_counts))
    assert abs(rep.final_objective - rep1.final_objective) <= 1e-9 * abs(rep1.final_objective)
    beta = geo.from_x([t.cpu().numpy() for t in betas])
    b1 = beta1.cpu().numpy()
    assert np.linalg.norm(beta - b1) <= 1e-8 * np.linalg.norm(b1)
    found = sh.gather_support(betas, geo, grid.comm)
    np.testing.assert_array_equal(found, np.sort(idx))


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_dropin_solve_matches_single_gpu(P):
    """sharded.solve(b, mask, config): the reference calling convention
    (NumPy b, Mask, default lambda) over P emulated ranks == fl.solve."""
    from paper_2502_04217_b200 import workloads

    inst = workloads.c3_bragg(32, seed=0)
    mask = fl.Mask.from_bool(inst.flags, fl.GridShape(inst.dims))
    b = fl.observe(inst.beta_true, mask) + inst.noise
    beta1, rep1 = fl.solve(b, mask, fl.IpmConfig(tol=1e-8))
    beta, rep = sh.solve(b, mask, fl.IpmConfig(tol=1e-8), comm=sh.LocalComm(P))
    assert isinstance(beta, np.ndarray) and beta.shape == beta1.shape
    assert abs(rep.lam - rep1.lam) <= 1e-12 * rep1.lam
    assert rep.status == rep1.status == "converged" and rep.iterations == rep1.iterations
    assert all(abs(x - y) <= 1 for x, y in zip(rep.krylov_counts, rep1.krylov_counts))
    assert abs(rep.final_objective - rep1.final_objective) <= 1e-9 * abs(rep1.final_objective)
    assert np.linalg.norm(beta - beta1) <= 1e-8 * np.linalg.norm(beta1)


def test_sharded_dropin_solve_nccl_world_size_one():
    """The DistComm route (object broadcast, NCCL gather) at world size 1."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2502_04217_b200 import workloads

    inst = workloads.c4_const(32)
    mask = fl.Mask.from_bool(inst.flags, fl.GridShape(inst.dims))
    b = fl.observe(inst.beta_true, mask) + inst.noise
    beta1, rep1 = fl.solve(b, mask, fl.IpmConfig(lam=inst.lam))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        beta, rep = sh.solve(b, mask, fl.IpmConfig(lam=inst.lam))
    finally:
        dist.destroy_process_group()
    assert rep.krylov_counts == rep1.krylov_counts
    assert abs(rep.final_objective - rep1.final_objective) <= 1e-9 * abs(rep1.final_objective)
    assert np.linalg.norm(beta - beta1) <= 1e-8 * np.linalg.norm(beta1)


@pytest.mark.parametrize("P,dims", [(2, (128, 64, 64)), (4, (128, 128, 64))])
def test_sharded_device_inputs_weak_scaling_shapes(P, dims):
    """The bench's N = 2 / 4 weak-scaling grids are non-cubic ((2s, s, s),
    (2s, 2s, s)): device-generated slab inputs and the sharded solve against
    the single-GPU solve of the same recipe on the same grid."""
    import torch

    from paper_2502_04217_b200 import workloads
    from paper_2502_04217_b200.masking import BraggMask, restrict

    shape = fl.GridShape(dims)
    idx, val = workloads.c4_spikes(shape.n)
    mask = BraggMask(shape)
    beta_t = torch.zeros(shape.n, dtype=torch.float64, device="cuda")
    beta_t[torch.from_numpy(idx).cuda()] = torch.from_numpy(val).cuda()
    x = fl.synthesize(beta_t, shape)
    d0, d1, d2 = dims
    workloads.noisy_embed_device(x, mask.on_device().bits, dims, (0, 0, 0), (d1 * d2, d2, 1), 0)
    b = restrict(x, mask)
    beta1, rep1 = fl.solve(b, mask, fl.IpmConfig(lam=0.5))
    grid = sh.ShardedGrid(dims, sh.LocalComm(P), exchange="peer")
    prob, idx2, _, lam = sh.c4_problem_device(grid, noise_seed=0)
    betas, rep = sh.sharded_solve(prob, lam, fl.IpmConfig(lam=lam))
    assert rep.status == rep1.status == "converged" and abs(rep.iterations - rep1.iterations) <= 1
    assert abs(rep.final_objective - rep1.final_objective) <= 1e-9 * abs(rep1.final_objective)
    beta = grid.geo.from_x([t.cpu().numpy() for t in betas])
    assert np.linalg.norm(beta - beta1.cpu().numpy()) <= 1e-8 * float(beta1.norm())
    np.testing.assert_array_equal(sh.gather_support(betas, grid.geo, grid.comm), np.sort(idx))


def _shared_gpu_ok():
    """Two processes may share the GPU (compute mode Default)."""
    import subprocess

    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=compute_mode", "--format=csv,noheader", "-i", "0"],
                             capture_output=True, text=True, timeout=30).stdout.strip()
    except Exception:  # nvidia-smi missing: assume the default mode
        return True
    return out in ("", "Default")


@pytest.mark.skipif(not _shared_gpu_ok(), reason="GPU compute mode forbids two processes")
def test_peer_exchange_across_processes():
    """The peer exchange over REAL CUDA-IPC buffers between two processes
    (tests/_ipc_worker.py: a gloo group, both processes on cuda:0, one slab
    rank each; no kernel waits on another rank): the handle all-gather and
    open (DistComm.peer_buffers), the cross-process stores of the transposing
    exchange kernels and the drained-stream barrier give bitwise the results
    of two emulated ranks in one process, for the gram, the residual pass,
    the KKT apply and a whole sharded IPM solve."""
    import os
    import socket
    import subprocess
    import sys

    from conftest import REPO

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(REPO, "tests", "_ipc_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)
    assert res["world"] == 2
    assert all(res["bitwise_vs_emulated"].values()), res
    assert all(res["a2a_bitwise_vs_peer"].values()), res
    assert res["norm_equal"]
    assert res["solve"] == res["solve_emulated"] and res["solve"][0] == "converged", res
    assert res["gram_vs_single_gpu"] <= 1e-12
    d = res["dropin_vs_single_gpu"]  # sharded.solve (reference arguments on root) vs fl.solve on one GPU
    assert d["status"] == ["converged", "converged"] and d["iterations"][0] == d["iterations"][1]
    assert all(abs(a - b) <= 1 for a, b in zip(*d["krylov"]))
    assert d["objective_rel"] <= 1e-9 and d["beta_rel_l2"] <= 1e-8


@pytest.mark.skipif(not _shared_gpu_ok(), reason="GPU compute mode forbids two processes")
def test_bench_multiprocess_path_gloo():
    """The bench's N > 1 code path (torchrun, one process per rank, one JSON
    line from rank 0: sharded matvec + sharded C4-recipe solve) with two
    processes sharing the GPU over a gloo group -- what the driver's scaling
    run executes over NCCL, checked end to end (timings meaningless here)."""
    import os
    import socket
    import subprocess
    import sys

    from conftest import REPO

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(REPO, "bench.py"),
           "--dist-backend", "gloo", "--size", "64", "--steps", "2", "--warmup", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]  # rank 0 alone prints
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["value"] > 0 and res["config"]["parallelism"] == "slab x2"
    sol = res["solve"]
    assert sol["status"] == "converged" and sol["support_exact"] and sol["exchange"] == "peer", sol
