#!/usr/bin/env python
"""Benchmark of the B200 hot path: KKT matvecs/s at 512^3 + full IPM solve.

Metric (BASELINE.json): "IPM solve time & KKT matvecs/s at 512^3 (HBM GB/s
% of peak)".  One *step* is one condensed KKT matvec K (d_beta, d_z)
(newton_system.py:148-152) on the C4 configuration -- a 512^3 grid with the
Bragg-peak punch mask -- i.e. one fused gram (5 HBM passes) + epilogue.

  value     matvecs/s over all ranks, device-resident inputs, CUDA events.
  e2e       same metric through the public drop-in call
            ``newton_system.apply_kkt(d_beta, d_z, diag, mask)`` with pinned
            HOST direction vectors: H2D of (d_beta, d_z) and D2H of
            (top, bottom) inside the timed region every step.
  roofline  dominant pass of the matvec, algorithmic bytes / its CUDA-event
            time, against MEASURED_PEAKS.json's HBM copy bandwidth;
            ``roofline_operator`` does the same for the whole matvec
            (120.125 B/voxel).
  solve     full IPM solve of the C4 recipe at 512^3 (lambda = 0.5), device
            time and end-to-end time with NumPy in / NumPy out.
  cpu_baseline  the CPU oracle (NumPy/SciPy restatement of the reference,
            oracle/) timed on this host: one matvec at 512^3.

``--impl reference`` times the reference's CPU path (the oracle port; the
reference is pure Python and not present on the GPU box) on the same
workload and prints the same JSON line with "impl": "reference".
Inputs are 4 GiB per matvec (> 126 MB L2), so no explicit L2 flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "KKT matvecs/s at 512^3 (condensed K apply, C4 Bragg-punched grid)"
UNIT = "matvec/s"
PASS_NAMES_3D = ["synth_axis0", "synth_axis1", "gram_mid_axis2", "analyze_axis1", "analyze_axis0",
                 "kkt_epilogue"]
# operator order B (fl_kkt_order 1: 3D with axes 0 and 2 of 512): contiguous axis
# first and last, the fused mask pass on axis 0, the epilogue fused into the last pass
PASS_NAMES_3D_B = ["synth_axis2", "synth_axis1", "gram_mask_axis0", "analyze_axis1",
                   "analyze_axis2_kkt_epilogue"]


def pass_layout(plan_handle, n: int, ndim: int):
    """(names, minimum HBM bytes) of each launch of one KKT matvec as executed.

    Transform passes read + write one fp64 grid (16 B/voxel; the fused mask
    pass also reads the n/8-byte bitmask); the KKT epilogue reads d_beta, d_z,
    sigma1, sigma2 and writes top, bottom.  Order A runs it as a separate pass
    that also reads g (56 B/voxel; 136.125 executed B/voxel per matvec); order B
    fuses it into the last analysis (16 + 40 = 56 B/voxel for that pass), which
    executes exactly the 120.125 B/voxel operator model of SURVEY 8d.
    """
    from paper_2502_04217_b200 import _lib

    if ndim == 1:
        return ["gram_mask_axis0", "kkt_epilogue"], [16.125 * n, 56.0 * n]
    mid = 16.0 * n + n / 8.0
    if ndim == 3 and _lib.lib().fl_kkt_order(plan_handle) == 1:
        return PASS_NAMES_3D_B, [16.0 * n, 16.0 * n, mid, 16.0 * n, 56.0 * n]
    names = ([f"synth_axis{a}" for a in range(ndim - 1)] + [f"gram_mid_axis{ndim - 1}"]
             + [f"analyze_axis{a}" for a in range(ndim - 2, -1, -1)] + ["kkt_epilogue"])
    return names, [16.0 * n] * (ndim - 1) + [mid] + [16.0 * n] * (ndim - 1) + [56.0 * n]


def l2_note(size: int, per: str = "") -> str:
    """The L2 statement of the config: the four input grids (d_beta, d_z, sigma1, sigma2) per step."""
    gib = 4 * 8 * size ** 3 / 2 ** 30
    if gib * 2 ** 30 > 126e6:
        return f"inputs {gib:g} GiB{per} per step > 126 MB L2 (no flush needed)"
    return f"inputs {gib * 1024:g} MiB{per} per step fit the 126 MB L2 (small check size; not a bench config)"


def bench_config(size: int, world: int) -> dict:
    """The workload description, identical in both arms (b200 and reference)."""
    if world <= 1:
        return {"workload": f"C4: {size}^3 Bragg-punched grid (15.1% missing), one condensed KKT matvec "
                            "K (d_beta, d_z) per step (newton_system.py:148-152)",
                "n": size ** 3, "parallelism": "1 GPU",
                "l2": l2_note(size)}
    dims = weak_dims(world, size)
    return {"workload": f"slab-sharded condensed KKT matvec, global grid {list(dims)} ({size}^3 voxels per "
                        "GPU, weak scaling), one matvec per step",
            "n": int(np.prod(dims)), "parallelism": f"slab x{world}",
            "l2": l2_note(size, " per GPU")}


def measured_peak_hbm():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region.

    NVML (nvidia-ml-py) polled from a thread every 5 ms; falls back to
    ``nvidia-smi -lms 100`` when NVML is unavailable.
    """

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self._stop = None
        self._thread = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self._stop = threading.Event()

            def poll():
                while not self._stop.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        self.samples.append((float(mhz), int(rs)))
                    except Exception:
                        pass
                    self._stop.wait(0.005)

            self._thread = threading.Thread(target=poll, daemon=True)
            self._thread.start()
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no NVML samples"]}
        sm = [m for m, _ in self.samples]
        reasons = sorted({k for _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "samples": len(sm),
                "reasons": reasons, "source": "nvml"}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def c4_mask(side: int):
    from paper_2502_04217_b200 import workloads
    return workloads.bragg_flags(side)


def make_kkt_inputs(side: int, seed: int = 0):
    """Device-resident interior state diagonals and a direction at side^3."""
    import torch
    from paper_2502_04217_b200 import _dev, _lib

    n = side ** 3
    gen = torch.Generator(device="cuda").manual_seed(seed)
    s1, s2, nu1, nu2 = (torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) + 0.4
                        for _ in range(4))
    sig1, sig2 = _dev.empty(n), _dev.empty(n)
    _lib.call("fl_barrier_diagonals", n, _dev.ptr(s1), _dev.ptr(s2), _dev.ptr(nu1), _dev.ptr(nu2),
              _dev.ptr(sig1), _dev.ptr(sig2), None, None, None, None, _dev.stream())
    del s1, s2, nu1, nu2
    d = torch.randn(2 * n, dtype=torch.float64, device="cuda", generator=gen)
    return sig1, sig2, d


def run_b200(args, rank: int, world: int):
    import torch
    import torch.distributed as dist

    import paper_2502_04217_b200 as fl
    from paper_2502_04217_b200 import _dev, _lib
    from paper_2502_04217_b200.newton_system import BarrierDiagonals, apply_kkt

    side = args.size
    n = side ** 3
    dims = (side,) * 3
    shape = fl.GridShape(dims)
    flags = c4_mask(side)
    mask = fl.Mask.from_bool(flags, shape)
    dm = mask.on_device()
    plan = _dev.plan_for(dims)
    sig1, sig2, d = make_kkt_inputs(side, seed=rank)
    top, bot = _dev.empty(n), _dev.empty(n)
    s = _dev.stream()
    L = _lib.lib()

    def matvec():
        _lib.check(L.fl_kkt_apply(plan.handle, _dev.ptr(dm.bits), _dev.ptr(sig1), _dev.ptr(sig2),
                                  _dev.ptr(d[:n]), _dev.ptr(d[n:]), _dev.ptr(top), _dev.ptr(bot),
                                  None, s))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        matvec()
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            matvec()
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = world * args.steps / (ms_max / 1e3)

    # per-pass split (live CUDA events between passes)
    names, alg = pass_layout(plan.handle, n, len(dims))
    npass = len(names)
    acc = np.zeros(npass)
    reps = max(3, min(10, args.steps))
    buf = (__import__("ctypes").c_double * 8)()
    cnt = __import__("ctypes").c_int()
    for _ in range(reps):
        _lib.call("fl_kkt_apply_profiled", plan.handle, _dev.ptr(dm.bits), _dev.ptr(sig1), _dev.ptr(sig2),
                  _dev.ptr(d[:n]), _dev.ptr(d[n:]), _dev.ptr(top), _dev.ptr(bot), buf,
                  __import__("ctypes").byref(cnt), s)
        acc += np.array(buf[:npass])
    pass_ms = acc / reps
    peak, peak_src = measured_peak_hbm()
    passes = [{"name": names[i], "ms": round(float(pass_ms[i]), 4),
               "alg_bytes": alg[i], "GBps": round(alg[i] / pass_ms[i] / 1e6, 1),
               "frac": round(alg[i] / pass_ms[i] / 1e6 / peak, 4)} for i in range(npass)]
    dom = int(np.argmax(pass_ms))
    op_bytes = sum(alg)
    op_gbps = op_bytes / (ms_per_step * 1e6)
    traffic = None
    try:  # ncu dram bytes per launch of the same kernel, committed under profiles/
        with open(os.path.join(REPO, "profiles", "r02_traffic.json")) as fh:
            if side == 512:  # the capture of the operator order this plan runs
                tj = json.load(fh)
                key = "kernels_order_b" if names == PASS_NAMES_3D_B else "kernels"
                traffic = tj.get(key, {}).get(names[dom])
    except Exception:
        traffic = None
    roofline = {"bound": "hbm", "kernel": names[dom], "achieved": round(alg[dom] / pass_ms[dom] / 1e6, 1),
                "peak": peak, "unit": "GB/s", "frac": round(alg[dom] / pass_ms[dom] / 1e6 / peak, 4),
                "traffic": traffic, "peak_source": peak_src,
                "alg_bytes_per_launch": alg[dom]}
    model_bytes = 120.125 * n  # SURVEY 8d operator model (epilogue fused)
    op_gbps = model_bytes / (ms_per_step * 1e6)
    roofline_op = {"bound": "hbm", "achieved": round(op_gbps, 1), "peak": peak, "unit": "GB/s",
                   "frac": round(op_gbps / peak, 4), "alg_bytes_per_matvec": model_bytes,
                   "bytes_per_voxel": 120.125, "executed_bytes_per_voxel": op_bytes / n,
                   "executed_GBps": round(op_bytes / (ms_per_step * 1e6), 1)}
    clock = clocks.summary()

    # e2e (headline): the drop-in call exactly as a reference caller makes it --
    # NumPy d_beta, d_z and a NumPy BarrierDiagonals (newton_system.py:148-152;
    # the caller's diag comes from barrier_diagonals(NumPy ...)), so sigma1 and
    # sigma2 go up every call too: 4n doubles up, 2n down per step.
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    np_db, np_dz = d[:n].cpu().numpy(), d[n:].cpu().numpy()
    diag_np = BarrierDiagonals(sig1.cpu().numpy(), sig2.cpu().numpy(), None, None, None, None)

    def e2e_run(db_, dz_, diag_, reps):
        checksum = 0.0
        for _ in range(2):  # warm the pinned host-allocator cache
            out_top, out_bot = apply_kkt(db_, dz_, diag_, mask)
            del out_top, out_bot
        barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            out_top, out_bot = apply_kkt(db_, dz_, diag_, mask)  # returns host (NumPy) arrays
            checksum += float(out_top[0]) + float(out_bot[-1])  # consume, then drop
            del out_top, out_bot
        barrier()
        return time.perf_counter() - t0

    e2e_s = e2e_run(np_db, np_dz, diag_np, e2e_steps)
    e2e = {"value": round(world * e2e_steps / e2e_s, 3), "unit": UNIT,
           "h2d_bytes_per_step": 4 * n * 8, "d2h_bytes_per_step": 2 * n * 8, "steps": e2e_steps,
           "api": "newton_system.apply_kkt(NumPy d_beta, NumPy d_z, NumPy BarrierDiagonals, mask) -> NumPy"}
    del np_db, np_dz, diag_np
    # secondary: pinned host direction vectors, diagonals already on the device
    diag = BarrierDiagonals(sig1, sig2, None, None, None, None)
    h_db = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_dz = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_db.copy_(d[:n])
    h_dz.copy_(d[n:])
    e2e_p = e2e_run(h_db, h_dz, diag, e2e_steps)
    del h_db, h_dz
    e2e_pinned = {"value": round(world * e2e_steps / e2e_p, 3), "unit": UNIT,
                  "h2d_bytes_per_step": 2 * n * 8, "d2h_bytes_per_step": 2 * n * 8, "steps": e2e_steps,
                  "api": "newton_system.apply_kkt(pinned host d_beta, d_z; device-resident diagonals)"}

    del d, top, bot, sig1, sig2
    torch.cuda.empty_cache()
    solve_info = None
    other = None
    passes_1024 = None
    if not args.no_solve:
        solve_info = run_solve(args.solve_size, barrier)
        other = run_other_solves(barrier)
        if not args.no_c5:
            other["C5 1024^3 Bragg, lambda=0.5, ONE GPU"] = run_c5(barrier)
            try:  # the C5 axis length: per-pass table of one 1024^3 matvec
                passes_1024 = per_pass_table(1024)
            except Exception as exc:  # report, never hide
                passes_1024 = {"error": repr(exc)[:300]}
    roofline["operator"] = roofline_op
    return dict(value=value, ms_per_step=ms_per_step, roofline=roofline,
                passes=passes, clocks=clock, e2e=e2e, e2e_pinned=e2e_pinned, solve=solve_info, other=other,
                passes_1024=passes_1024,
                gpu_launches=args.steps * npass)


def per_pass_table(side: int, reps: int = 5):
    """Per-pass CUDA-event times of one KKT matvec at side^3 (fl_kkt_apply_profiled),
    device-resident inputs, Bragg mask built on the device."""
    import ctypes

    import torch

    import paper_2502_04217_b200 as fl
    from paper_2502_04217_b200 import _dev, _lib
    from paper_2502_04217_b200.masking import BraggMask

    n = side ** 3
    shape = fl.GridShape((side,) * 3)
    dm = BraggMask(shape).on_device()
    plan = _dev.plan_for(shape.dims)
    sig1, sig2, d = make_kkt_inputs(side, seed=7)
    top, bot = _dev.empty(n), _dev.empty(n)
    buf = (ctypes.c_double * 8)()
    cnt = ctypes.c_int()
    names, alg = pass_layout(plan.handle, n, 3)
    acc = np.zeros(len(names))
    for i in range(reps + 2):
        _lib.call("fl_kkt_apply_profiled", plan.handle, _dev.ptr(dm.bits), _dev.ptr(sig1), _dev.ptr(sig2),
                  _dev.ptr(d[:n]), _dev.ptr(d[n:]), _dev.ptr(top), _dev.ptr(bot), buf, ctypes.byref(cnt),
                  _dev.stream())
        if i >= 2:
            acc += np.array(buf[:len(names)])
    ms = acc / reps
    peak, _ = measured_peak_hbm()
    del sig1, sig2, d, top, bot, dm
    torch.cuda.empty_cache()
    return {"size": side, "matvec_ms": round(float(ms.sum()), 3), "matvec_per_s": round(1e3 / float(ms.sum()), 2),
            "operator_frac": round(120.125 * n / (float(ms.sum()) * 1e6) / peak, 4),
            "passes": [{"name": names[i], "ms": round(float(ms[i]), 4),
                        "GBps": round(alg[i] / ms[i] / 1e6, 1), "frac": round(alg[i] / ms[i] / 1e6 / peak, 4)}
                       for i in range(len(names))]}


def weak_dims(world: int, side: int = 512):
    """Global grid with side^3 voxels per GPU: N=2 -> (2s, s, s), 4 -> (2s, 2s, s),
    8 -> (2s, 2s, 2s) (= C5, 1024^3 at s = 512); other N -> (N s, s, s)."""
    return {1: (side,) * 3, 2: (2 * side, side, side), 4: (2 * side, 2 * side, side),
            8: (2 * side,) * 3}.get(world, (world * side, side, side))


def run_sharded(args, comm, barrier, max_ms):
    """Slab-sharded KKT matvec over comm.world ranks (real or emulated), device-timed and e2e."""
    import torch

    from paper_2502_04217_b200 import _dev, _lib
    from paper_2502_04217_b200 import sharded as sh

    dims = weak_dims(comm.world, args.size)
    grid = sh.ShardedGrid(dims, comm)
    geo = grid.geo
    nl = geo.n_local
    bits = [grid.ops[0].bits(sh.bragg_y_flags(geo, r)) for r in comm.ranks]
    sig1, sig2, ds = [], [], []
    for r in comm.ranks:
        a, b_, d = make_kkt_inputs_n(nl, seed=r)
        sig1.append(a)
        sig2.append(b_)
        ds.append(d)
    tops = [_dev.empty(nl) for _ in comm.ranks]
    bots = [_dev.empty(nl) for _ in comm.ranks]

    def matvec():
        sh.kkt_apply(grid, bits, sig1, sig2, [d[:nl] for d in ds], [d[nl:] for d in ds], tops, bots)

    for _ in range(args.warmup):
        matvec()
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            matvec()
        e1.record(stream)
        barrier()
    ms = max_ms(e0.elapsed_time(e1))
    # e2e: host slabs in, host slabs out, per rank
    h_d = [torch.empty(2 * nl, dtype=torch.float64, pin_memory=True) for _ in comm.ranks]
    for h, d in zip(h_d, ds):
        h.copy_(d)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dd = [h.to("cuda", non_blocking=True) for h in h_d]
        sh.kkt_apply(grid, bits, sig1, sig2, [d[:nl] for d in dd], [d[nl:] for d in dd], tops, bots)
        outs = [(t.cpu(), b_.cpu()) for t, b_ in zip(tops, bots)]
    barrier()
    e2e_s = max_ms((time.perf_counter() - t0) * 1e3) / 1e3
    del outs, h_d
    if hasattr(comm, "release_peer_buffers"):
        comm.release_peer_buffers()
    return dict(dims=dims, ms=ms, clocks=clocks.summary(),
                e2e=e2e_steps * comm.world / e2e_s, e2e_steps=e2e_steps, n_local=nl,
                launches=args.steps * (10 + 4) * len(comm.ranks))


def run_sharded_solve(args, comm, barrier, max_ms):
    """Full slab-sharded IPM solve of the C4/C5 recipe at the weak-scaling grid
    (N=8: 1024^3 = C5), inputs generated on the devices in slab layout
    (sharded.c4_problem_device).  Reports solve seconds (max over ranks),
    IPM / Krylov counts, objective and exact-support recovery; at 1024^3 the
    objective is compared with the single-GPU C5 solve of the same input
    (tests/golden/solve_c5_1gpu.json)."""
    import torch

    import paper_2502_04217_b200 as fl
    from paper_2502_04217_b200 import sharded as sh

    dims = weak_dims(comm.world, args.size)
    torch.cuda.empty_cache()
    grid = sh.ShardedGrid(dims, comm)
    barrier()
    t0 = time.perf_counter()
    prob, idx, _, lam = sh.c4_problem_device(grid, noise_seed=0)
    barrier()
    gen_s = max_ms((time.perf_counter() - t0) * 1e3) / 1e3
    torch.cuda.reset_peak_memory_stats()
    t0 = time.perf_counter()
    betas, rep = sh.sharded_solve(prob, lam, fl.IpmConfig(lam=lam, tol=1e-8))
    barrier()
    solve_s = max_ms((time.perf_counter() - t0) * 1e3) / 1e3
    found = sh.gather_support(betas, grid.geo, comm)
    out = {"dims": list(dims), "status": rep.status, "lambda": lam, "ipm_iterations": rep.iterations,
           "krylov": rep.krylov_counts, "total_krylov": rep.total_krylov, "solve_s": round(solve_s, 4),
           "final_objective": rep.final_objective,
           "support_exact": bool(np.array_equal(found, np.sort(idx))), "n_support": int(found.size),
           "input_generation_s": round(gen_s, 3),
           "device_peak_GB_rank0": round(torch.cuda.max_memory_allocated() / 1e9, 1),
           "exchange": grid.exchange,
           "note": "inputs generated on the devices in slab layout; solve_s = sharded IPM loop, "
                   "max over ranks (host-synchronised, perf_counter)"}
    ref_path = os.path.join(REPO, "tests", "golden", "solve_c5_1gpu.json")
    if tuple(dims) == (1024, 1024, 1024) and os.path.exists(ref_path):
        with open(ref_path) as fh:
            ref = json.load(fh)
        out["vs_single_gpu"] = {
            "objective_1gpu": ref["final_objective"],
            "objective_rel_diff": abs(rep.final_objective - ref["final_objective"]) / abs(ref["final_objective"]),
            "ipm_iterations_1gpu": ref["ipm_iterations"], "krylov_1gpu": ref["krylov"]}
    del betas, prob
    if hasattr(comm, "release_peer_buffers"):
        comm.release_peer_buffers()
    del grid
    torch.cuda.empty_cache()
    return out


def make_kkt_inputs_n(n: int, seed: int = 0):
    import torch
    from paper_2502_04217_b200 import _dev, _lib

    gen = torch.Generator(device="cuda").manual_seed(seed)
    s1, s2, nu1, nu2 = (torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) + 0.4
                        for _ in range(4))
    sig1, sig2 = _dev.empty(n), _dev.empty(n)
    _lib.call("fl_barrier_diagonals", n, _dev.ptr(s1), _dev.ptr(s2), _dev.ptr(nu1), _dev.ptr(nu2),
              _dev.ptr(sig1), _dev.ptr(sig2), None, None, None, None, _dev.stream())
    del s1, s2, nu1, nu2
    return sig1, sig2, torch.randn(2 * n, dtype=torch.float64, device="cuda", generator=gen)


def _solve_instance(inst, barrier, reps_warm=1, ista=False):
    """Cold + warm device solves and one NumPy-in/NumPy-out solve of a recipe instance."""
    import torch

    import paper_2502_04217_b200 as fl

    shape = fl.GridShape(inst.dims)
    mask = fl.Mask.from_bool(inst.flags, shape)
    bt = torch.from_numpy(inst.beta_true).cuda()
    b = fl.observe(bt, mask)
    b += torch.from_numpy(inst.noise).cuda()
    cfg = fl.IpmConfig(lam=inst.lam, tol=1e-8)
    barrier()
    t0 = time.perf_counter()
    beta, rep = fl.solve(b, mask, cfg)
    barrier()
    cold = time.perf_counter() - t0
    warm = []
    for _ in range(reps_warm):
        del beta
        t0 = time.perf_counter()
        beta, rep = fl.solve(b, mask, cfg)
        barrier()
        warm.append(time.perf_counter() - t0)
    cross = None
    if ista:
        # independent first-order oracle at full size: the
        # unguarded GPU ISTA must reach the IPM objective within 1e-6
        from paper_2502_04217_b200 import diagnostics as dg

        t0 = time.perf_counter()
        try:
            ref, iters = dg.ista_solve(b, mask, rep.lam, tol=1e-10, max_iters=3000, max_n=None)
            o_ipm = fl.lasso_objective(beta, b, mask, rep.lam)
            o_ista = fl.lasso_objective(ref, b, mask, rep.lam)
            same = bool(np.array_equal(dg.classify_support(beta).active, dg.classify_support(ref).active))
            cross = {"ista_iterations": iters, "ista_s": round(time.perf_counter() - t0, 3),
                     "ipm_objective": o_ipm, "ista_objective": o_ista,
                     "rel_diff": abs(o_ipm - o_ista) / abs(o_ista), "same_support": same}
            del ref
        except Exception as exc:  # report, never hide
            cross = {"error": repr(exc)[:300]}
    b_host = b.cpu().numpy()
    del b, bt, beta
    torch.cuda.empty_cache()
    barrier()
    e2e_runs = []
    for _ in range(2):  # steady state: the first call also pins the host staging
        beta_h = None
        t0 = time.perf_counter()
        beta_h, rep2 = fl.solve(b_host, mask, cfg)
        e2e_runs.append(time.perf_counter() - t0)
    e2e_s = min(e2e_runs)
    true_support = np.flatnonzero(inst.beta_true)
    found = np.flatnonzero(np.abs(beta_h) > 1e-6 * np.max(np.abs(beta_h)))
    return {"status": rep.status, "lambda": rep.lam, "ipm_iterations": rep.iterations,
            "krylov": rep.krylov_counts, "total_krylov": rep.total_krylov,
            "device_s_cold": round(cold, 4), "device_s": round(min(warm), 4), "e2e_s": round(e2e_s, 4),
            "e2e_s_first": round(e2e_runs[0], 4),
            "final_objective": rep.final_objective,
            "support_exact": bool(np.array_equal(found, true_support)), "n_support": int(found.size),
            **({"ista_crosscheck": cross} if ista else {})}


def run_solve(side: int, barrier):
    """Full IPM solve of the C4 recipe (lambda 0.5) at side^3."""
    from paper_2502_04217_b200 import workloads

    out = _solve_instance(workloads.c4_const(side), barrier, ista=True)
    out["config"] = f"C4 recipe {side}^3, lambda=0.5, tol=1e-8"
    # solve-level byte rate, lower bound: only the PCG iterations' traffic
    # (248 B/voxel each: 5-pass gram + fused update + p-update, DESIGN 4.2)
    pcg_bytes = out["total_krylov"] * 248.0 * side ** 3
    out["pcg_bytes_model"] = pcg_bytes
    out["achieved_GBps_lower_bound"] = round(pcg_bytes / out["device_s"] / 1e9, 1)
    return out


def run_other_solves(barrier):
    """Solve times of the other BASELINE configs (C1 1D 4096, C2 2048^2, C3 256^3)."""
    from paper_2502_04217_b200 import workloads

    res = {}
    for name, mk in (("C1 1D 4096 lambda=0.3", lambda: workloads.c1_1d(seed=0)),
                     ("C2 2048^2 block-punched, default lambda", lambda: workloads.c2_2d(seed=0)),
                     ("C3 256^3 Bragg-punched, default lambda", lambda: workloads.c3_bragg(256, seed=0))):
        try:
            res[name] = _solve_instance(mk(), barrier, reps_warm=2)
        except Exception as exc:  # report, never hide, a failing config
            res[name] = {"error": repr(exc)[:300]}
    return res


def run_c5(barrier):
    """C5 (1024^3, constant amplitudes, lambda 0.5) on ONE GPU: the solver's
    device footprint is 20 n doubles = 172 GB (SURVEY sizes C5 for 8 GPUs)."""
    import torch

    import paper_2502_04217_b200 as fl
    from paper_2502_04217_b200 import workloads

    torch.cuda.empty_cache()
    try:
        # inputs generated on the device (workloads.c4_const_device: device Bragg
        # mask, the recipe's spikes, device-RNG noise): no n-sized host arrays
        t0 = time.perf_counter()
        mask, b, idx, _, lam = workloads.c4_const_device(1024)
        gen_s = time.perf_counter() - t0
        b_host = b.cpu().numpy()  # the NumPy-in / NumPy-out drop-in call below
        del b
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        cfg = fl.IpmConfig(lam=lam, tol=1e-8)
        barrier()
        t0 = time.perf_counter()
        beta, rep = fl.solve(b_host, mask, cfg)
        e2e_s = time.perf_counter() - t0
        found = np.flatnonzero(np.abs(beta) > 1e-6 * np.max(np.abs(beta)))
        out = {"status": rep.status, "lambda": rep.lam, "ipm_iterations": rep.iterations,
               "krylov": rep.krylov_counts, "total_krylov": rep.total_krylov,
               "device_s": round(rep.wall_time, 4), "e2e_s_first": round(e2e_s, 4),
               "final_objective": rep.final_objective,
               "support_exact": bool(np.array_equal(found, np.sort(idx))),
               "n_support": int(found.size),
               "device_peak_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1),
               "input_generation_s": round(gen_s, 3),
               "note": "inputs generated on the GPU; device_s = IPM loop (host-synchronised, "
                       "perf_counter); e2e = NumPy in/out, first call"}
        del beta, b_host, mask
    except Exception as exc:  # report, never hide
        out = {"error": repr(exc)[:300]}
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# CPU arms (the oracle port of the reference; test infrastructure only)
# ---------------------------------------------------------------------------

def cpu_inputs(side: int, seed: int = 0):
    from oracle import fftlasso_oracle as orc

    n = side ** 3
    rng = np.random.default_rng(seed)
    s = [rng.random(n) + 0.4 for _ in range(4)]
    diag = orc.diagonals(*s)
    del s
    mask = orc.make_mask((side,) * 3, flags=c4_mask(side))
    return diag, mask, rng.standard_normal(n), rng.standard_normal(n)


def cpu_matvec_seconds(side: int, reps: int, warmup: int, budget_s: float):
    from oracle import fftlasso_oracle as orc

    diag, mask, db, dz = cpu_inputs(side)
    for _ in range(warmup):
        orc.kkt_apply(db, dz, diag, mask)
    times = []
    t_start = time.perf_counter()
    for _ in range(reps):
        t0 = time.perf_counter()
        orc.kkt_apply(db, dz, diag, mask)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    return times


def cpu_cores() -> int:
    cap = os.environ.get("FFTLASSO_THREADS")
    return max(1, int(cap)) if cap else (os.cpu_count() or 1)


def cpu_solve_seconds(inst, reps: int):
    """Full CPU solves of a recipe instance with the oracle port (the reference's
    own bench harness times solve() with perf_counter, cli.py:117-122)."""
    from oracle import fftlasso_oracle as orc

    om = orc.make_mask(inst.dims, flags=inst.flags)
    b = orc.observe(inst.beta_true, om) + inst.noise
    times, rep = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        _, rep = orc.solve(b, om, orc.OConfig(lam=inst.lam, tol=1e-8))
        times.append(time.perf_counter() - t0)
    return {"solve_s": round(statistics.median(times), 4), "runs": reps, "status": rep.status,
            "ipm_iterations": rep.iterations, "krylov": rep.krylov_counts, "final_objective": rep.final_objective}


def run_reference(args):
    times = cpu_matvec_seconds(args.size, args.steps, min(args.warmup, 1), args.ref_budget)
    per = sum(times) / len(times)
    value = 1.0 / per
    sample = (f"{len(times)} of {args.steps} requested steps (time cap {args.ref_budget:.0f} s), "
              f"each one oracle kkt_apply at {args.size}^3; warmup {min(args.warmup, 1)}")
    solves = {}
    if not args.no_solve:
        from paper_2502_04217_b200 import workloads

        for name, mk, reps in (("C1 1D 4096 lambda=0.3", lambda: workloads.c1_1d(seed=0), 3),
                               ("C2 2048^2 block-punched, default lambda", lambda: workloads.c2_2d(seed=0), 1)):
            try:
                solves[name] = cpu_solve_seconds(mk(), reps)
            except Exception as exc:  # report, never hide
                solves[name] = {"error": repr(exc)[:300]}
        solves["C3 256^3 Bragg-punched, default lambda"] = {
            "not_run": "~8 min of CPU; the reference's own converged solve took 494.7 s on 8 threads "
                       "(tests/golden/solve_c3_256.json cpu_seconds)"}
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(times), "warmup": min(args.warmup, 1),
        "ms_per_step": round(per * 1e3, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.size, int(os.environ.get("WORLD_SIZE", "1"))),
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": cpu_cores(), "kind": "port",
                         "sample": sample,
                         "impl": "NumPy/SciPy oracle port of fftlasso (the reference is pure Python and "
                                 "cannot travel to the GPU box); pocketfft workers = cores"},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_solves": solves, "host": host_info(),
    }
    print(json.dumps(line), flush=True)


def host_info() -> dict:
    info = {"cpu_count": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    info["model"] = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--solve-size", type=int, default=512)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the 1024^3 single-GPU solve")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-budget", type=float, default=150.0)
    ap.add_argument("--emulate", type=int, default=0,
                    help="run the sharded (N>1) code path with P emulated ranks on one GPU")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded path (torch.distributed + NCCL) even at one rank")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend of the N > 1 path; gloo (host-side collectives, ranks may "
                         "share a GPU) only checks the multi-process code path -- its timings mean nothing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return

    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    gloo = args.dist_backend == "gloo"
    if gloo:  # ranks may share GPUs (a multi-process check of this code path on one box)
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1 or args.emulate > 1 or args.sharded:
        from paper_2502_04217_b200 import sharded as sh

        if world > 1 or args.sharded:
            if gloo:
                dist.init_process_group("gloo")
                comm = sh.DistComm()
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
                comm = sh.DistComm(device=torch.device("cuda", local))

            def barrier():
                torch.cuda.synchronize()
                dist.barrier()
                torch.cuda.synchronize()

            def max_ms(v):
                t = torch.tensor([v], dtype=torch.float64, device="cpu" if gloo else "cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                return float(t.item())
        else:
            comm = sh.LocalComm(args.emulate)

            def barrier():
                torch.cuda.synchronize()

            def max_ms(v):
                return v
        res = run_sharded(args, comm, barrier, max_ms)
        solve = None
        if not args.no_solve:
            try:
                solve = run_sharded_solve(args, comm, barrier, max_ms)
            except Exception as exc:  # report, never hide
                solve = {"error": repr(exc)[:300]}
        P = comm.world
        if rank == 0:
            n_all = res["n_local"] * P
            value = P * args.steps / (res["ms"] / 1e3)
            peak, peak_src = measured_peak_hbm()
            line = {
                "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms"] / args.steps, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": bench_config(args.size, P),
                "emulated": isinstance(comm, sh.LocalComm),
                "exchange": "5 HBM passes + 2 slab transposes (peer stores over NVLink, or NCCL all-to-all) "
                            "+ epilogue per matvec",
                "roofline": {"bound": "hbm", "achieved": round(120.125 * n_all / P / (res["ms"] / args.steps * 1e6), 1),
                             "peak": peak, "unit": "GB/s",
                             "frac": round(120.125 * n_all / P / (res["ms"] / args.steps * 1e6) / peak, 4),
                             "traffic": None, "peak_source": peak_src,
                             "note": "per-GPU algorithmic bytes of the matvec (120.125 B/voxel) / step time"},
                "cpu_baseline": None,
                "e2e": {"value": round(res["e2e"], 3), "unit": UNIT,
                        "h2d_bytes_per_step": 2 * n_all * 8, "d2h_bytes_per_step": 2 * n_all * 8,
                        "steps": res["e2e_steps"], "api": "sharded.kkt_apply with pinned host slabs"},
                "clocks": res["clocks"], "gpu_launches": res["launches"], "solve": solve,
            }
            print(json.dumps(line), flush=True)
        if dist.is_available() and dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()
        return
    res = run_b200(args, rank, world)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            times = cpu_matvec_seconds(args.size, 2, 1, 60.0)
            cpu = {"value": round(len(times) / sum(times), 5), "unit": UNIT, "cores": cpu_cores(), "kind": "port",
                   "sample": f"{len(times)} oracle kkt_apply at {args.size}^3 after 1 warm-up "
                             f"(NumPy/SciPy, pocketfft workers={cpu_cores()})"}
        line = {
            "metric": METRIC, "value": round(res["value"], 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_per_step"], 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": bench_config(args.size, world),
            "roofline": res["roofline"],
            "passes": res["passes"], "cpu_baseline": cpu, "e2e": res["e2e"], "e2e_pinned": res["e2e_pinned"],
            "clocks": res["clocks"],
            "gpu_launches": res["gpu_launches"], "solve": res["solve"], "solves_other_configs": res["other"],
            "passes_1024": res["passes_1024"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
