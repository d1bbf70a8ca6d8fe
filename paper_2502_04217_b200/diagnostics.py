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

* ``scaling_trajectory_check`` / ``ScalingReport`` -- the barrier-scaling
  probe over the tail of an IPM trajectory (diagnostics.py:234-322), with the
  barrier diagonals and the per-class ratio ranges computed on the GPU; the
  trajectory is the list of states ``solve``'s observer receives (a fresh
  snapshot per iteration, as the reference passes).

The dense-matrix probes of the reference (``densify``, the dense spectrum
probe) are O(n^2)-O(n^3) test tooling outside the hot path; the GPU test
suite runs them from the oracle (``oracle/fftlasso_oracle.py``) on the
observer's snapshots of GPU solves (reference acceptance criteria 5-6).
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
    "ScalingReport",
    "scaling_trajectory_check",
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


@dataclass
class ScalingReport:
    """Observed barrier scaling ratios over the tail of a trajectory (diagnostics.py:234-268)."""

    band: tuple
    iterations_checked: int
    lambda1_times_mu: tuple
    sigma1_over_mu_pos: tuple
    sigma2_times_mu_pos: tuple
    sigma1_times_mu_neg: tuple
    sigma2_over_mu_neg: tuple
    sigma1_times_mu_zero: tuple
    sigma2_times_mu_zero: tuple
    sigma_product_active: tuple
    in_band: bool

    def to_dict(self) -> dict:
        out = {"record": "scaling", "band": list(self.band), "iterations_checked": self.iterations_checked}
        for k in ("lambda1_times_mu", "sigma1_over_mu_pos", "sigma2_times_mu_pos", "sigma1_times_mu_neg",
                  "sigma2_over_mu_neg", "sigma1_times_mu_zero", "sigma2_times_mu_zero", "sigma_product_active"):
            out[k] = list(getattr(self, k))
        out["in_band"] = self.in_band
        return out


def scaling_trajectory_check(states, support: SupportClassification | None = None,
                             band: tuple = (1.0 / 50.0, 50.0), tail: int = 5) -> ScalingReport:
    """Barrier-diagonal growth rates over the last ``tail`` iterates (diagnostics.py:271-322).

    Expected by class of the final solution: sigma1 ~ mu, sigma2 ~ 1/mu on
    positive indices (mirrored on negative ones), both ~ 1/mu on zero
    indices, lambda1 ~ 1/mu everywhere, sigma1 sigma2 of order one on the
    active set.  mu is each state's duality measure.  The diagonals and the
    ratio ranges are computed on the GPU (NumPy or CUDA states).
    """
    import torch

    from .newton_system import barrier_diagonals

    if not states:
        raise ValueError("empty trajectory")
    window = states[-tail:]
    if support is None:
        support = classify_support(window[-1].beta)
    dev = _dev.device()
    cls = [torch.as_tensor(np.asarray(a, dtype=np.int64), device=dev)
           for a in (support.positive, support.negative, support.zero, support.active)]
    pos, neg, zero, active = cls
    acc = [[] for _ in range(8)]
    for st in window:
        mu = st.duality_measure()
        d = barrier_diagonals(_dev.to_dev(st.s1), _dev.to_dev(st.s2), _dev.to_dev(st.nu1), _dev.to_dev(st.nu2))
        s1, s2 = d.sigma1, d.sigma2
        for i, v in enumerate((d.lambda1 * mu, s1[pos] / mu, s2[pos] * mu, s1[neg] * mu, s2[neg] / mu,
                               s1[zero] * mu, s2[zero] * mu, s1[active] * s2[active])):
            acc[i].append(v)
    ranges = []
    for chunk in acc:
        v = torch.cat(chunk)
        ranges.append((1.0, 1.0) if v.numel() == 0 else (float(v.min()), float(v.max())))
    lo, hi = band
    return ScalingReport(band=tuple(band), iterations_checked=len(window), lambda1_times_mu=ranges[0],
                         sigma1_over_mu_pos=ranges[1], sigma2_times_mu_pos=ranges[2],
                         sigma1_times_mu_neg=ranges[3], sigma2_over_mu_neg=ranges[4],
                         sigma1_times_mu_zero=ranges[5], sigma2_times_mu_zero=ranges[6],
                         sigma_product_active=ranges[7],
                         in_band=all(lo <= r[0] and r[1] <= hi for r in ranges))
