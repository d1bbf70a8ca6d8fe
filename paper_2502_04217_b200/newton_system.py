"""Condensed Newton (KKT) systems, B200 path (reference newton_system.py).

Same public functions and dataclasses as the reference.  The elementwise
kernels (csrc/fl_vec.cu) evaluate every formula in NumPy's order without
FMA contraction, so diagonals, right-hand sides, the preconditioner and the
recovered blocks are bitwise equal to the reference on equal inputs; the
gram inside ``apply_kkt`` is the fused FFT operator (tolerance-equal).

Block structure (newton_system.py:1-36):

    K = [ G + Lam1   Lam2 ]      P = [ I + Lam1   Lam2 ]
        [ Lam2       Lam1 ]          [ Lam2       Lam1 ]
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import UnsupportedShapeError
from .masking import Mask, embed_device

__all__ = [
    "BarrierDiagonals",
    "KktRhs",
    "CondensedSolution",
    "barrier_diagonals",
    "newton_rhs",
    "apply_kkt",
    "apply_precond_inverse",
    "apply_precond_kkt",
    "recover_eliminated",
]


@dataclass(frozen=True)
class BarrierDiagonals:
    """Diagonal data of K and P (newton_system.py:60-69); device tensors."""

    sigma1: object
    sigma2: object
    lambda1: object
    lambda2: object
    dvec: object
    bvec: object


def _vec(x, n=None):
    return _dev.to_dev(x, n)


def barrier_diagonals(s1, s2, nu1, nu2) -> BarrierDiagonals:
    """sigma = nu/s and the derived diagonals (newton_system.py:72-91).

    Raises InteriorViolationError when any input is <= 0 or non-finite.
    """
    host = not _dev.is_device(s1)
    s1d = _vec(s1)
    n = s1d.numel()
    s2d, n1d, n2d = _vec(s2, n), _vec(nu1, n), _vec(nu2, n)
    outs = [_dev.empty(n) for _ in range(6)]
    _lib.call("fl_barrier_diagonals", n, *(_dev.ptr(t) for t in (s1d, s2d, n1d, n2d)),
              *(_dev.ptr(t) for t in outs), _dev.stream())
    return BarrierDiagonals(*(_dev.out(t, host) for t in outs))


@dataclass(frozen=True)
class KktRhs:
    """All six block residuals and the condensed pair (newton_system.py:94-110)."""

    r1: object
    r2: object
    r3: object
    r4: object
    r5: object
    r6: object
    r_beta: object
    r_c: object


def fl_state(st) -> _lib.FlState:
    return _lib.FlState(*(_dev.ptr(getattr(st, f)) for f in
                          ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2")))


def newton_rhs(state, b, mask: Mask, lam: float) -> KktRhs:
    """Residuals of the barrier KKT system (newton_system.py:113-145)."""
    from .ipm import as_device_state

    host = not _dev.is_device(state.beta)
    st = as_device_state(state)
    n = mask.shape.n
    diag = barrier_diagonals(st.s1, st.s2, st.nu1, st.nu2)
    bd = _vec(b, mask.n_observed)
    bhat = embed_device(bd, mask)
    plan = _dev.plan_for(mask.shape.dims)
    g = _dev.empty(n)
    dm = mask.on_device()
    _lib.call("fl_residual_adjoint", plan.handle, _dev.ptr(dm.bits), _dev.ptr(bhat),
              _dev.ptr(st.beta), _dev.ptr(g), _dev.stream())
    outs = [_dev.empty(n) for _ in range(8)]
    fs = fl_state(st)
    _lib.call("fl_newton_rhs", n, _lib.ctypes.byref(fs), _dev.ptr(g), _dev.ptr(diag.sigma1),
              _dev.ptr(diag.sigma2), float(lam), float(st.mu), *(_dev.ptr(t) for t in outs),
              _dev.stream())
    return KktRhs(*(_dev.out(t, host) for t in outs))


_STREAM_MIN = 1 << 20  # host-data calls at least this large stream through PCIe in chunks
_STREAM_CHUNKS = 8
_copy_streams: dict = {}


def _host_tensor(x, n):
    import torch

    if isinstance(x, torch.Tensor):
        t = x.detach().reshape(-1)
        return t if t.dtype == torch.float64 and t.is_contiguous() else t.to(torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1)))


def _apply_kkt_streamed(d_beta, d_z, diag: BarrierDiagonals, mask: Mask):
    """apply_kkt for host inputs: PCIe transfers overlapped with the work.

    d_beta goes up first and the gram runs on it while d_z -- and sigma1,
    sigma2 when the diagonals are host arrays too (a NumPy caller's
    BarrierDiagonals) -- stream up in chunks; each chunk's epilogue (top
    needs g, d_z and the sigmas, bottom d_beta, d_z and the sigmas) runs as
    soon as its inputs land and its results stream back on a third stream,
    so device->host traffic overlaps host->device traffic (PCIe is full
    duplex).  Pageable NumPy sources are staged through pinned chunks by
    worker threads (``_dev.upload_chunks``).  Same kernels as the device
    path, results bitwise equal.
    """
    import torch

    n = mask.shape.n
    hb, hz = _host_tensor(d_beta, n), _host_tensor(d_z, n)
    if hb.numel() != n or hz.numel() != n:
        raise UnsupportedShapeError(f"direction blocks must have {n} entries")
    dev = _dev.device()
    if dev.index not in _copy_streams:
        _copy_streams[dev.index] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    h2d, d2h = _copy_streams[dev.index]
    comp = torch.cuda.current_stream()
    db, dz, top, bot = (_dev.empty(n) for _ in range(4))
    sig_host = [not _dev.is_device(x) for x in (diag.sigma1, diag.sigma2)]
    g1 = _dev.empty(n) if sig_host[0] else _vec(diag.sigma1, n)
    g2 = _dev.empty(n) if sig_host[1] else _vec(diag.sigma2, n)
    out_t = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out_b = torch.empty(n, dtype=torch.float64, pin_memory=True)
    step = -(-n // _STREAM_CHUNKS)
    step += step % 2  # 16-byte epilogue accesses
    bounds = [(a, min(n, a + step)) for a in range(0, n, step)]
    h2d.wait_stream(comp)  # the device buffers were allocated on the compute stream
    # upload order: all of d_beta (the gram needs it whole), then per chunk
    # d_z and the host sigmas; one event per (d_beta) and per chunk
    jobs = [[(hb, db, 0, n)]]
    for a, b in bounds:
        grp = [(hz, dz, a, b)]
        for is_host, src, dst in zip(sig_host, (diag.sigma1, diag.sigma2), (g1, g2)):
            if is_host:
                grp.append((_host_tensor(src, n), dst, a, b))
        jobs.append(grp)
    events = _dev.upload_chunks(jobs, h2d)
    plan = _dev.plan_for(mask.shape.dims)
    dm = mask.on_device()
    comp.wait_event(events[0])
    _lib.call("fl_gram", plan.handle, _dev.ptr(dm.bits), _dev.ptr(db), _dev.ptr(top), _dev.stream())
    sz = 8  # bytes per double
    for (a, b), e in zip(bounds, events[1:]):
        comp.wait_event(e)
        off = a * sz
        _lib.call("fl_kkt_epilogue", b - a, ctypes.c_void_p(top.data_ptr() + off),
                  ctypes.c_void_p(db.data_ptr() + off), ctypes.c_void_p(dz.data_ptr() + off),
                  ctypes.c_void_p(g1.data_ptr() + off), ctypes.c_void_p(g2.data_ptr() + off),
                  ctypes.c_void_p(bot.data_ptr() + off), None, _dev.stream())
        done = torch.cuda.Event()
        done.record(comp)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            out_t[a:b].copy_(top[a:b], non_blocking=True)
            out_b[a:b].copy_(bot[a:b], non_blocking=True)
    d2h.synchronize()
    for t in (db, dz, top, bot, g1, g2):  # keep the caching allocator stream-safe
        t.record_stream(h2d)
        t.record_stream(d2h)
    return out_t.numpy(), out_b.numpy()


def apply_kkt(d_beta, d_z, diag: BarrierDiagonals, mask: Mask):
    """(top, bottom) = K (d_beta, d_z) (newton_system.py:148-152), one fused operator.

    Host inputs (NumPy or CPU tensors) at n >= 2^20 take the streamed path:
    PCIe uploads, the operator and the downloads overlap chunk by chunk.
    """
    host = not _dev.is_device(d_beta)
    n = mask.shape.n
    if host and not _dev.is_device(d_z) and n % 2 == 0 and n >= _STREAM_MIN:
        return _apply_kkt_streamed(d_beta, d_z, diag, mask)
    db, dz = _vec(d_beta, n), _vec(d_z, n)
    top, bot = _dev.empty(n), _dev.empty(n)
    plan = _dev.plan_for(mask.shape.dims)
    dm = mask.on_device()
    g1, g2 = _vec(diag.sigma1, n), _vec(diag.sigma2, n)
    _lib.call("fl_kkt_apply", plan.handle, _dev.ptr(dm.bits), _dev.ptr(g1), _dev.ptr(g2), _dev.ptr(db), _dev.ptr(dz), _dev.ptr(top), _dev.ptr(bot),
              None, _dev.stream())
    return _dev.out(top, host), _dev.out(bot, host)


def apply_precond_inverse(r_beta, r_c, diag: BarrierDiagonals):
    """Closed-form P^{-1} (newton_system.py:155-159)."""
    host = not _dev.is_device(r_beta)
    rb = _vec(r_beta)
    n = rb.numel()
    rc = _vec(r_c, n)
    top, bot = _dev.empty(n), _dev.empty(n)
    g1, g2 = _vec(diag.sigma1, n), _vec(diag.sigma2, n)
    _lib.call("fl_precond_apply", n, _dev.ptr(g1), _dev.ptr(g2), _dev.ptr(rb),
              _dev.ptr(rc), _dev.ptr(top), _dev.ptr(bot), _dev.stream())
    return _dev.out(top, host), _dev.out(bot, host)


def apply_precond_kkt(d_beta, d_z, diag: BarrierDiagonals, mask: Mask):
    """P^{-1} K (newton_system.py:162-165)."""
    host = not _dev.is_device(d_beta)
    top, bot = apply_kkt(_vec(d_beta), _vec(d_z), diag, mask)
    t, b = apply_precond_inverse(top, bot, diag)
    return _dev.out(t, host), _dev.out(b, host)


@dataclass(frozen=True)
class CondensedSolution:
    """Full 6-block direction in the symmetrized convention (newton_system.py:168-181)."""

    d_beta: object
    d_z: object
    d_s1: object
    d_s2: object
    d_y1: object
    d_y2: object


def recover_eliminated(d_beta, d_z, rhs: KktRhs, diag: BarrierDiagonals) -> CondensedSolution:
    """Back-substitute multipliers and slacks (newton_system.py:184-196)."""
    host = not _dev.is_device(d_beta)
    db = _vec(d_beta)
    n = db.numel()
    dz = _vec(d_z, n)
    rs = [_vec(getattr(rhs, f), n) for f in ("r3", "r4", "r5", "r6")]
    outs = [_dev.empty(n) for _ in range(4)]
    g1, g2 = _vec(diag.sigma1, n), _vec(diag.sigma2, n)
    _lib.call("fl_recover_eliminated", n, _dev.ptr(g1), _dev.ptr(g2),
              *(_dev.ptr(t) for t in rs), _dev.ptr(db), _dev.ptr(dz), *(_dev.ptr(t) for t in outs),
              _dev.stream())
    ds1, ds2, dy1, dy2 = (_dev.out(t, host) for t in outs)
    return CondensedSolution(_dev.out(db, host), _dev.out(dz, host), ds1, ds2, dy1, dy2)
