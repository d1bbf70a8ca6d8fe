"""Solver cross-checks on the B200 path (reference diagnostics.py:112-360).

* ``soft_threshold`` -- one elementwise kernel with NumPy's sign / maximum
  conventions, bitwise equal to ``np.sign(x) * np.maximum(|x| - t, 0)``.
* ``classify_support`` / ``SupportClassification`` -- the support partition
  the parity tests grade on (SURVEY §8c hazard H4).
* ``ista_solve`` -- the first-order oracle the reference uses to cross-check
  IPM objectives, with every iteration on the GPU: the fused gram (2d-1 HBM
  passes) plus one fused step kernel (gradient, shrinkage, max-norm
  displacement).  The reference refuses n > 4096 (``ISTA_DIM_GUARD``); the
  default here is the same, and ``max_n=None`` lifts the guard so the GPU
  ISTA can check IPM objectives at sizes where no CPU or dense oracle runs
  (SURVEY §8f item 2).

The dense-matrix probes of the reference (``densify``, spectrum and scaling
probes) are test tooling built on O(n^2) dense matrices, outside the hot
path; IPM state snapshots for such probes come from ``solve``'s observer.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import IterationLimitError
from .masking import Mask, embed_device

__all__ = [
    "ISTA_DIM_GUARD",
    "ISTA_ITER_CAP",
    "SupportClassification",
    "classify_support",
    "soft_threshold",
    "ista_solve",
]

ISTA_DIM_GUARD = 4096
ISTA_ITER_CAP = 10**6


@dataclass(frozen=True)
class SupportClassification:
    """Indices by solution sign (diagnostics.py:112-126)."""

    positive: np.ndarray
    negative: np.ndarray
    zero: np.ndarray
    threshold: float

    @property
    def active(self) -> np.ndarray:
        return np.union1d(self.positive, self.negative)

    @property
    def n_active(self) -> int:
        return int(self.positive.size + self.negative.size)


def classify_support(beta, threshold: float | None = None) -> SupportClassification:
    """Positive / negative / numerically-zero sets (diagnostics.py:129-142).

    Default threshold ``1e-6 * max|beta|``.  Host bookkeeping on the final
    coefficients (a CUDA tensor is copied back once).
    """
    if _dev.is_device(beta):
        beta = beta.detach().cpu().numpy()
    v = np.asarray(beta, dtype=np.float64).reshape(-1)
    if threshold is None:
        threshold = 1e-6 * (float(np.max(np.abs(v))) if v.size else 0.0)
    t = float(threshold)
    return SupportClassification(np.flatnonzero(v > t), np.flatnonzero(v < -t),
                                 np.flatnonzero((v >= -t) & (v <= t)), t)


def soft_threshold(x, t: float):
    """Proximity operator of ``t * ||.||_1`` (diagnostics.py:325-328), on the GPU."""
    host = not _dev.is_device(x)
    shape = np.shape(x) if host else tuple(x.shape)
    v = _dev.to_dev(x, None)
    out = _dev.empty(v.numel())
    _lib.call("fl_soft_threshold", v.numel(), _dev.ptr(v), float(t), _dev.ptr(out), _dev.stream())
    res = _dev.out(out, host)
    return res.reshape(shape)


def ista_solve(b, mask: Mask, lam: float, tol: float = 1e-10,
               max_iters: int = ISTA_ITER_CAP, max_n: int | None = ISTA_DIM_GUARD):
    """Iterative soft thresholding (diagnostics.py:331-360) -> (beta, iterations).

    Unit step (the gram of orthonormal rows has norm <= 1); stops when the
    max-norm displacement drops to ``tol``.  Raises ``IterationLimitError``
    past ``max_iters`` and ``ValueError`` when ``n > max_n`` (the reference's
    guard; pass ``max_n=None`` for the unguarded GPU cross-check).
    """
    n = mask.shape.n
    if max_n is not None and n > max_n:
        raise ValueError(f"ISTA oracle guard: n {n} > {max_n}")
    host = not _dev.is_device(b)
    bv = _dev.to_dev(b, mask.n_observed, "observed vector")
    plan = _dev.plan_for(mask.shape.dims)
    dm = mask.on_device()
    s = _dev.stream()
    xi = embed_device(bv, mask)                       # observe_adjoint(b)
    _lib.call("fl_analyze", plan.handle, _dev.ptr(xi), _dev.ptr(xi), s)
    beta, nxt, g = _dev.zeros(n), _dev.empty(n), _dev.empty(n)
    step = ctypes.c_double()
    for k in range(1, int(max_iters) + 1):
        _lib.call("fl_gram", plan.handle, _dev.ptr(dm.bits), _dev.ptr(beta), _dev.ptr(g), s)
        _lib.call("fl_ista_step", n, _dev.ptr(beta), _dev.ptr(g), _dev.ptr(xi), float(lam),
                  _dev.ptr(nxt), ctypes.byref(step), s)
        beta, nxt = nxt, beta
        if step.value <= tol:
            return _dev.out(beta, host), k
    raise IterationLimitError(f"ISTA did not reach tol={tol:.1e} within {max_iters} iterations")
