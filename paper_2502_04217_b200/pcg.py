"""Preconditioned conjugate gradients, B200 path (reference pcg.py).

Two entry points:

* ``pcg_solve(apply_op, apply_prec, rhs, config)`` -- the reference's
  matrix-free plug-in interface (pcg.py:57-127): callables on flat vectors.
  Vectors live on the GPU; dots and the x/r/p recurrences are
  libfftlasso_b200 kernels.  With NumPy ``rhs`` the callables receive and may
  return NumPy arrays (drop-in for the reference's callers); with a CUDA
  tensor they receive CUDA tensors.
* ``kkt_pcg(...)`` -- the solver's hot loop: PCG on the condensed KKT system
  fully inside the C library (``fl_pcg_kkt``), fused matvec + fused update;
  the iteration loop runs on the device (a CUDA graph with a WHILE node), so a
  whole PCG solve is one graph launch and one host round trip.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from .errors import NumericalBreakdownError

__all__ = ["PcgConfig", "PcgResult", "pcg_solve"]

MAX_ITERS_CAP = 5000  # pcg.py:19


@dataclass(frozen=True)
class PcgConfig:
    """Stopping control (pcg.py:22-45)."""

    abs_tol: float = 1e-12
    rel_tol: float = 0.0
    max_iters: int | None = None
    record_history: bool = False

    def __post_init__(self):
        if self.abs_tol < 0 or self.rel_tol < 0:
            raise ValueError("tolerances must be nonnegative")
        if self.abs_tol == 0 and self.rel_tol == 0:
            raise ValueError("abs_tol and rel_tol cannot both be zero")

    def iteration_limit(self, dim: int) -> int:
        if self.max_iters is not None:
            return int(self.max_iters)
        return min(10 * dim, MAX_ITERS_CAP)


@dataclass
class PcgResult:
    solution: object
    iterations: int
    converged: bool
    residual_norm: float
    residual_history: list[float] | None = field(default=None)


def _dot(a, b) -> float:
    out = ctypes.c_double()
    _lib.call("fl_dot", a.numel(), _dev.ptr(a), _dev.ptr(b), ctypes.byref(out), _dev.stream())
    return out.value


def pcg_solve(apply_op, apply_prec, rhs, config: PcgConfig = PcgConfig()) -> PcgResult:
    """Solve K x = rhs by PCG from x0 = 0 (pcg.py:57-127)."""
    host = not _dev.is_device(rhs)
    b = _dev.to_dev(rhs)
    dim = b.numel()
    limit = config.iteration_limit(dim)

    def call(fn, v):
        res = fn(v.cpu().numpy() if host else v)
        return _dev.to_dev(res, dim, "operator output")

    x = _dev.zeros(dim)
    r = b.clone()
    z = call(apply_prec, r)
    rho = _dot(r, z)
    if not math.isfinite(rho) or rho < 0:
        raise NumericalBreakdownError(f"preconditioner produced r'P^{{-1}}r = {rho}")
    norm0 = math.sqrt(rho)
    threshold = config.abs_tol + config.rel_tol * norm0
    history = [norm0] if config.record_history else None
    if norm0 <= threshold:
        return PcgResult(_dev.out(x, host), 0, True, norm0, history)
    p = z.clone()
    norm = norm0
    s = _dev.stream()
    for k in range(1, limit + 1):
        kp = call(apply_op, p)
        curvature = _dot(p, kp)
        if not math.isfinite(curvature) or curvature <= 0:
            raise NumericalBreakdownError(
                f"nonpositive curvature p'Kp = {curvature} at iteration {k}")
        alpha = rho / curvature
        _lib.call("fl_axpy", dim, alpha, _dev.ptr(p), _dev.ptr(x), s)
        _lib.call("fl_axpy", dim, -alpha, _dev.ptr(kp), _dev.ptr(r), s)
        z = call(apply_prec, r)
        rho_next = _dot(r, z)
        if not math.isfinite(rho_next) or rho_next < 0:
            raise NumericalBreakdownError(f"r'P^{{-1}}r = {rho_next} at iteration {k}")
        norm = math.sqrt(rho_next)
        if history is not None:
            history.append(norm)
        if norm <= threshold:
            return PcgResult(_dev.out(x, host), k, True, norm, history)
        _lib.call("fl_xpby", dim, _dev.ptr(z), rho_next / rho, _dev.ptr(p), s)
        rho = rho_next
    return PcgResult(_dev.out(x, host), limit, False, norm, history)


def kkt_pcg(plan, dmask, sigma1, sigma2, rhs2n, x2n, work, config: PcgConfig):
    """Device-resident PCG on the condensed KKT system (fl_pcg_kkt).

    ``rhs2n``/``x2n`` are 2n CUDA tensors [beta-block; z-block]; ``work`` has
    ``fl_pcg_work_doubles(n)`` entries.  Returns a PcgResult whose solution
    is ``x2n``.
    """
    n = plan.n
    res = _lib.FlPcgResult()
    limit = config.iteration_limit(2 * n)
    hist = None
    if config.record_history:
        hist = np.zeros(limit + 1, dtype=np.float64)
    _lib.call("fl_pcg_kkt", plan.handle, _dev.ptr(dmask.bits), _dev.ptr(sigma1), _dev.ptr(sigma2),
              _dev.ptr(rhs2n), _dev.ptr(x2n), _dev.ptr(work), float(config.abs_tol),
              float(config.rel_tol), int(limit), ctypes.byref(res),
              hist.ctypes.data_as(ctypes.c_void_p) if hist is not None else None,
              int(limit + 1) if hist is not None else 0, _dev.stream())
    history = None
    if hist is not None:
        history = hist[: int(res.iterations) + 1].tolist()
    return PcgResult(x2n, int(res.iterations), bool(res.converged), float(res.residual_norm), history)
