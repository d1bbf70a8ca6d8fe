"""Primal-dual interior-point driver, B200 path (reference ipm.py).

Same algorithm, parameters, records and return values as the reference.
``solve`` keeps the whole iterate on the GPU and runs each iteration as

    barrier diagonals -> fused RHS -> device PCG (fl_pcg_kkt) ->
    fused back-substitution + fraction-to-boundary minima ->
    fused state update -> ONE residual transform A^T Z (b - A beta) ->
    fused KKT/barrier-residual assessment

so the data correlation r1 is computed once per iteration (the reference
recomputes the identical vector three times).  Host work is the
scalar control flow of ipm.py:439-469 on values read back from the device.
The public helpers (newton_direction, ipm_step, check_convergence, ...) keep
the reference's signatures; ``ipm_step`` calls ``newton_direction`` through
this module's globals, as the reference does.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import InteriorViolationError, NumericalBreakdownError, StalledError
from .masking import Mask, embed_device
from .newton_system import (
    BarrierDiagonals,
    KktRhs,
    barrier_diagonals,
    fl_state,
    newton_rhs,
)
from .pcg import PcgConfig, PcgResult, kkt_pcg

__all__ = [
    "IpmConfig",
    "IpmState",
    "IterationRecord",
    "SolveReport",
    "ConvergenceReport",
    "NewtonDirection",
    "default_penalty",
    "lasso_objective",
    "initial_state",
    "newton_direction",
    "ipm_step",
    "next_barrier",
    "check_convergence",
    "fraction_to_boundary",
    "solve",
]

FIELDS = ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2")


@dataclass(frozen=True)
class IpmConfig:
    """Solver parameters (ipm.py:55-82)."""

    lam: float | None = None
    tol: float = 1e-8
    max_iters: int = 200
    mu_init: float | None = None
    sigma_mu: float = 0.2
    mu_power: float = 1.5
    ftb_tau: float = 0.995
    gamma_centrality: float = 1e-4
    cg_tol: float = 1e-12
    cg_max_iters: int | None = None
    inner_slack: float = 10.0

    def __post_init__(self):
        if not 0.0 < self.sigma_mu < 1.0:
            raise ValueError("sigma_mu must lie in (0, 1)")
        if not 0.0 < self.ftb_tau < 1.0:
            raise ValueError("ftb_tau must lie in (0, 1)")
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")


def _min_of(t) -> float:
    out = ctypes.c_double()
    d = _dev.to_dev(t)
    _lib.call("fl_min", d.numel(), _dev.ptr(d), ctypes.byref(out), _dev.stream())
    return out.value


def _dot(a, b) -> float:
    out = ctypes.c_double()
    da, db = _dev.to_dev(a), _dev.to_dev(b)
    _lib.call("fl_dot", da.numel(), _dev.ptr(da), _dev.ptr(db), ctypes.byref(out), _dev.stream())
    return out.value


@dataclass
class IpmState:
    """All primal-dual iterates plus the barrier parameter (ipm.py:85-110).

    Fields are CUDA tensors (solver-internal states) or NumPy arrays (states
    built by host callers); every method works on both.
    """

    beta: object
    z: object
    s1: object
    s2: object
    y1: object
    y2: object
    nu1: object
    nu2: object
    mu: float

    @property
    def n(self) -> int:
        b = self.beta
        return int(b.numel() if hasattr(b, "numel") else np.asarray(b).size)

    def duality_measure(self) -> float:
        """(nu1's1 + nu2's2) / 2n, dots on the GPU (ipm.py:103-105)."""
        return float(_dot(self.nu1, self.s1) + _dot(self.nu2, self.s2)) / (2 * self.n)

    def assert_interior(self):
        for name in ("s1", "s2", "nu1", "nu2"):
            if _min_of(getattr(self, name)) <= 0.0:
                raise StalledError(f"{name} left the strict interior")

    def to_numpy(self) -> "IpmState":
        conv = (lambda v: v.cpu().numpy()) if _dev.is_device(self.beta) else np.asarray
        return IpmState(mu=self.mu, **{f: conv(getattr(self, f)) for f in FIELDS})


def as_device_state(state) -> IpmState:
    if _dev.is_device(state.beta):
        return state
    n = np.asarray(state.beta).size
    return IpmState(mu=state.mu, **{f: _dev.to_dev(getattr(state, f), n) for f in FIELDS})


@dataclass(frozen=True)
class ConvergenceReport:
    """Residuals of the exact (mu = 0) KKT conditions (ipm.py:113-125)."""

    stationarity: float
    dual_equality: float
    multiplier_gap: float
    primal: float
    complementarity: float
    max_residual: float
    converged: bool
    centrality_ok: bool
    duality_measure: float


@dataclass
class IterationRecord:
    iteration: int
    mu: float
    primal_inf: float
    dual_inf: float
    complementarity: float
    kkt_max: float
    krylov_iters: int
    alpha_primal: float
    alpha_dual: float
    pcg_residual: float
    centrality_ok: bool
    wall_time: float

    def to_dict(self) -> dict:
        """JSON record, same keys as ipm.py:143-158."""
        return {
            "record": "iteration",
            "iteration": self.iteration,
            "mu": self.mu,
            "primal_inf": self.primal_inf,
            "dual_inf": self.dual_inf,
            "complementarity": self.complementarity,
            "kkt_max": self.kkt_max,
            "krylov_iters": self.krylov_iters,
            "alpha_primal": self.alpha_primal,
            "alpha_dual": self.alpha_dual,
            "pcg_residual": self.pcg_residual,
            "centrality_ok": self.centrality_ok,
            "wall_time": self.wall_time,
        }


@dataclass
class SolveReport:
    status: str
    iterations: int
    lam: float
    tol: float
    records: list[IterationRecord]
    final_objective: float
    final_kkt: float
    final_mu: float
    wall_time: float

    @property
    def converged(self) -> bool:
        return self.status == "converged"

    @property
    def krylov_counts(self) -> list[int]:
        return [rec.krylov_iters for rec in self.records]

    @property
    def total_krylov(self) -> int:
        return sum(self.krylov_counts)

    def to_dict(self) -> dict:
        """JSON summary, same keys as ipm.py:185-197."""
        return {
            "record": "summary",
            "status": self.status,
            "iterations": self.iterations,
            "lambda": self.lam,
            "tol": self.tol,
            "final_objective": self.final_objective,
            "final_kkt": self.final_kkt,
            "final_mu": self.final_mu,
            "total_krylov": self.total_krylov,
            "wall_time": self.wall_time,
        }


# ---------------------------------------------------------------------------
# per-problem device data
# ---------------------------------------------------------------------------

class Problem:
    """Device-resident (plan, mask bits, embedded observations) of one instance."""

    def __init__(self, b, mask: Mask, scratch=None):
        self.mask = mask
        self.n = mask.shape.n
        self.plan = _dev.plan_for(mask.shape.dims)
        self.dmask = mask.on_device()
        # only the embedded b_hat stays resident: host observations are uploaded
        # into ``scratch`` (the solver's PCG work buffer) and embedded from there
        self.bhat = embed_device(_dev.to_dev(b, mask.n_observed, "observed vector", scratch=scratch), mask)

    def residual_adjoint(self, beta, out):
        """out = A^T Z (b_hat - A beta); beta None -> A^T b_hat."""
        _lib.call("fl_residual_adjoint", self.plan.handle, _dev.ptr(self.dmask.bits),
                  _dev.ptr(self.bhat), _dev.ptr(beta) if beta is not None else None,
                  _dev.ptr(out), _dev.stream())
        return out

    def default_penalty(self, scratch=None) -> float:
        g = self.residual_adjoint(None, scratch if scratch is not None else _dev.empty(self.n))
        m = ctypes.c_double()
        _lib.call("fl_max_abs", self.n, _dev.ptr(g), ctypes.byref(m), _dev.stream())
        return 0.1 * float(m.value)

    def objective(self, beta, lam: float, work) -> float:
        out = ctypes.c_double()
        _lib.call("fl_lasso_objective", self.plan.handle, _dev.ptr(self.dmask.bits),
                  _dev.ptr(self.bhat), _dev.ptr(beta), float(lam), _dev.ptr(work),
                  ctypes.byref(out), _dev.stream())
        return out.value

    def assess(self, st: IpmState, g, lam: float, mu: float, fs=None) -> _lib.FlAssess:
        a = _lib.FlAssess()
        fs = fl_state(st) if fs is None else fs
        _lib.call("fl_ipm_assess", self.n, ctypes.byref(fs), _dev.ptr(g), float(lam), float(mu),
                  ctypes.byref(a), _dev.stream())
        return a


def _conv_report(a: _lib.FlAssess, n: int, tol: float, gamma: float) -> ConvergenceReport:
    worst = max(a.stationarity, a.dual_equality, a.multiplier_gap, a.primal, a.complementarity)
    measure = float(a.dot_nu_s1 + a.dot_nu_s2) / (2 * n)
    return ConvergenceReport(
        stationarity=a.stationarity,
        dual_equality=a.dual_equality,
        multiplier_gap=a.multiplier_gap,
        primal=a.primal,
        complementarity=a.complementarity,
        max_residual=worst,
        converged=worst <= tol,
        centrality_ok=bool(a.min_product >= gamma * measure),
        duality_measure=measure,
    )


# ---------------------------------------------------------------------------
# public helpers (reference signatures)
# ---------------------------------------------------------------------------

def default_penalty(b, mask: Mask) -> float:
    """0.1 * max|observe_adjoint(b)| (ipm.py:204-206)."""
    return Problem(b, mask).default_penalty()


def lasso_objective(beta, b, mask: Mask, lam: float) -> float:
    """0.5 ||b - observe(beta)||^2 + lam ||beta||_1 (ipm.py:209-211)."""
    prob = Problem(b, mask)
    return prob.objective(_dev.to_dev(beta, prob.n), lam, _dev.empty(prob.n))


def initial_state(b, mask: Mask, lam: float, mu_init: float | None = None) -> IpmState:
    """beta=0, z=s=1, y=nu=lam/2, mu=lam/2 (ipm.py:214-238)."""
    if lam <= 0:
        raise ValueError("penalty must be positive")
    n = mask.shape.n
    st = IpmState(mu=lam / 2.0 if mu_init is None else float(mu_init),
                  **{f: _dev.empty(n) for f in FIELDS})
    fs = fl_state(st)
    _lib.call("fl_ipm_init", n, ctypes.byref(fs), float(lam), _dev.stream())
    return st if _dev.is_device(b) else st.to_numpy()


def check_convergence(state: IpmState, b, mask: Mask, lam: float,
                      tol: float, gamma: float = 1e-4) -> ConvergenceReport:
    """Exact KKT residuals and the centrality monitor (ipm.py:241-273)."""
    prob = Problem(b, mask)
    st = as_device_state(state)
    g = prob.residual_adjoint(st.beta, _dev.empty(prob.n))
    return _conv_report(prob.assess(st, g, lam, st.mu), prob.n, tol, gamma)


@dataclass(frozen=True)
class NewtonDirection:
    """Physical step for every block plus solve diagnostics (ipm.py:285-300)."""

    d_beta: object
    d_z: object
    d_s1: object
    d_s2: object
    d_y1: object
    d_y2: object
    d_nu1: object
    d_nu2: object
    krylov_iters: int
    pcg_residual: float
    rhs: KktRhs | None
    diag: BarrierDiagonals | None


def _pcg_config(config: IpmConfig) -> PcgConfig:
    return PcgConfig(abs_tol=config.cg_tol, max_iters=config.cg_max_iters)


def newton_direction(state: IpmState, b, mask: Mask, lam: float,
                     config: IpmConfig) -> NewtonDirection:
    """One Newton direction at the current mu (ipm.py:303-352)."""
    host = not _dev.is_device(state.beta)
    st = as_device_state(state)
    prob = Problem(b, mask)
    n = prob.n
    diag = barrier_diagonals(st.s1, st.s2, st.nu1, st.nu2)
    rhs = newton_rhs(st, b, mask, lam)
    rhs2n = _dev.empty(2 * n)
    rhs2n[:n].copy_(rhs.r_beta)
    rhs2n[n:].copy_(rhs.r_c)
    x = _dev.empty(2 * n)
    work = _dev.empty(_lib.lib().fl_pcg_work_doubles(n))
    res = kkt_pcg(prob.plan, prob.dmask, diag.sigma1, diag.sigma2, rhs2n, x, work, _pcg_config(config))
    if not res.converged:
        raise NumericalBreakdownError(
            f"PCG stalled at preconditioned residual {res.residual_norm:.3e} "
            f"after {res.iterations} iterations")
    outs = [_dev.empty(n) for _ in range(6)]
    fs = fl_state(st)
    _lib.call("fl_ipm_direction", n, ctypes.byref(fs), _dev.ptr(diag.sigma1), _dev.ptr(diag.sigma2),
              float(st.mu), _dev.ptr(x[:n]), _dev.ptr(x[n:]), *(_dev.ptr(t) for t in outs),
              _dev.stream())
    o = lambda t: _dev.out(t, host)  # noqa: E731
    if host:
        rhs = KktRhs(*(o(getattr(rhs, f)) for f in ("r1", "r2", "r3", "r4", "r5", "r6", "r_beta", "r_c")))
        diag = BarrierDiagonals(*(o(getattr(diag, f)) for f in
                                  ("sigma1", "sigma2", "lambda1", "lambda2", "dvec", "bvec")))
    return NewtonDirection(o(x[:n].clone()), o(x[n:].clone()), *(o(t) for t in outs),
                           krylov_iters=res.iterations, pcg_residual=res.residual_norm,
                           rhs=rhs, diag=diag)


def fraction_to_boundary(v, dv, tau: float) -> float:
    """Largest step in (0, 1] with v + alpha dv >= (1 - tau) v (ipm.py:355-361)."""
    vd = _dev.to_dev(v)
    dvd = _dev.to_dev(dv, vd.numel())
    out = ctypes.c_double()
    _lib.call("fl_ftb_ratio", vd.numel(), _dev.ptr(vd), _dev.ptr(dvd), ctypes.byref(out), _dev.stream())
    return _alpha_from_ratio(out.value, tau)


def _alpha_from_ratio(ratio: float, tau: float) -> float:
    if ratio == math.inf:  # no component shrinks
        return 1.0
    return min(1.0, tau * ratio)


def ipm_step(state: IpmState, b, mask: Mask, lam: float,
             config: IpmConfig) -> tuple[IpmState, NewtonDirection, float, float]:
    """One damped Newton step (ipm.py:364-394)."""
    host = not _dev.is_device(state.beta)
    direction = newton_direction(state, b, mask, lam, config)
    tau = max(config.ftb_tau, 1.0 - state.mu)
    alpha_p = min(fraction_to_boundary(state.s1, direction.d_s1, tau),
                  fraction_to_boundary(state.s2, direction.d_s2, tau))
    alpha_d = min(fraction_to_boundary(state.nu1, direction.d_nu1, tau),
                  fraction_to_boundary(state.nu2, direction.d_nu2, tau))
    if min(alpha_p, alpha_d) < 1e-12:
        raise StalledError(
            f"fraction-to-boundary step collapsed (alpha_p={alpha_p:.2e}, alpha_d={alpha_d:.2e})")
    n = state.n
    new = IpmState(mu=state.mu, **{f: _dev.to_dev(getattr(state, f), n).clone() for f in FIELDS})
    dirs = IpmState(mu=0.0, **{f: _dev.to_dev(getattr(direction, "d_" + f), n) for f in FIELDS})
    fs, fd = fl_state(new), fl_state(dirs)
    _lib.call("fl_ipm_update_explicit", n, ctypes.byref(fs), ctypes.byref(fd), float(alpha_p),
              float(alpha_d), _dev.stream())
    return (new.to_numpy() if host else new), direction, alpha_p, alpha_d


def next_barrier(mu: float, tol: float, config: IpmConfig) -> float:
    """Monotone barrier schedule with a superlinear tail (ipm.py:397-399)."""
    return max(tol / 10.0, min(config.sigma_mu * mu, mu ** config.mu_power))


# ---------------------------------------------------------------------------
# the solver
# ---------------------------------------------------------------------------

class Workspace:
    """Every device vector one solve needs: 19 n doubles (+ b_hat in Problem).

    g = A^T Z (b_hat - A beta) lives in the PCG work buffer's G p slot
    (work[4n:5n]): it is consumed by the Newton setup pass before the PCG
    loop overwrites that slot and recomputed after the state update, so the
    two never overlap in time.  20 n doubles = 160 B/voxel in total: 21.5 GB
    at 512^3, 172 GB at 1024^3 (C5 fits one 180 GB B200).
    """

    def __init__(self, n: int):
        self.state = IpmState(mu=0.0, **{f: _dev.empty(n) for f in FIELDS})
        self.sig1 = _dev.empty(n)
        self.sig2 = _dev.empty(n)
        self.x = _dev.empty(2 * n)
        self.work = _dev.empty(_lib.lib().fl_pcg_work_doubles(n))
        self.g = self.work[4 * n:5 * n]
        self.best_beta = _dev.empty(n)
        self.fs = fl_state(self.state)
        self.verdict = _dev.pinned(16)  # fl_ipm_newton_step's step record


def _fused_step(prob: Problem, ws: Workspace, mu: float, lam: float, config: IpmConfig):
    """ipm_step (ipm.py:364-394) with every vector op fused on the device.

    ``fl_ipm_newton_pcg`` is the front half of newton_direction: one pass for
    the barrier diagonals (interior check), the condensed RHS and the PCG
    start, then the device-looped PCG (ipm.py:303-332).
    """
    n = prob.n
    s = _dev.stream()
    pc = _pcg_config(config)
    out = _lib.FlPcgResult()
    _lib.call("fl_ipm_newton_pcg", prob.plan.handle, _dev.ptr(prob.dmask.bits), ctypes.byref(ws.fs),
              _dev.ptr(ws.g), float(lam), float(mu), _dev.ptr(ws.sig1), _dev.ptr(ws.sig2), _dev.ptr(ws.x),
              _dev.ptr(ws.work), float(pc.abs_tol), float(pc.rel_tol), int(pc.iteration_limit(2 * n)),
              ctypes.byref(out), s)
    res = PcgResult(ws.x, int(out.iterations), bool(out.converged), float(out.residual_norm), None)
    if not res.converged:
        raise NumericalBreakdownError(
            f"PCG stalled at preconditioned residual {res.residual_norm:.3e} "
            f"after {res.iterations} iterations")
    tau = max(config.ftb_tau, 1.0 - mu)
    ratios = (ctypes.c_double * 4)()
    db, dz = _dev.ptr(ws.x[:n]), _dev.ptr(ws.x[n:])
    _lib.call("fl_ipm_ratios", n, ctypes.byref(ws.fs), _dev.ptr(ws.sig1), _dev.ptr(ws.sig2),
              float(mu), db, dz, ratios, s)
    alpha_p = min(_alpha_from_ratio(ratios[0], tau), _alpha_from_ratio(ratios[1], tau))
    alpha_d = min(_alpha_from_ratio(ratios[2], tau), _alpha_from_ratio(ratios[3], tau))
    if min(alpha_p, alpha_d) < 1e-12:
        raise StalledError(
            f"fraction-to-boundary step collapsed (alpha_p={alpha_p:.2e}, alpha_d={alpha_d:.2e})")
    _lib.call("fl_ipm_update", n, ctypes.byref(ws.fs), _dev.ptr(ws.sig1), _dev.ptr(ws.sig2),
              float(mu), db, dz, float(alpha_p), float(alpha_d), s)
    return res, alpha_p, alpha_d


# True (default): the whole step is issued with one sync (the assessment's);
# False: a host sync after each stage (_fused_step) -- same kernels in the
# same order, bitwise the same iterates (tests flip this attribute).
_ASYNC_STEP = True


def _launch_step(prob: Problem, ws: Workspace, mu: float, lam: float, config: IpmConfig) -> None:
    """ipm_step (ipm.py:364-394) issued without waiting: PCG, step lengths and
    the state update run on the device; the verdict lands in ``ws.verdict``."""
    n = prob.n
    pc = _pcg_config(config)
    tau = max(config.ftb_tau, 1.0 - mu)
    _lib.call("fl_ipm_newton_step", prob.plan.handle, _dev.ptr(prob.dmask.bits), ctypes.byref(ws.fs),
              _dev.ptr(ws.g), float(lam), float(mu), float(tau), _dev.ptr(ws.sig1), _dev.ptr(ws.sig2),
              _dev.ptr(ws.x), _dev.ptr(ws.work), float(pc.abs_tol), float(pc.rel_tol),
              int(pc.iteration_limit(2 * n)), ws.verdict.data_ptr(), _dev.stream())


def _step_verdict(ws: Workspace):
    """Read the step record after the stream synchronised; raise as the
    synchronous path would (PCG breakdown / stall, collapsed step, interior)."""
    v = ws.verdict.tolist()
    status, k = int(v[8]), int(v[9])
    if status == 3:
        raise NumericalBreakdownError(f"nonpositive curvature p'Kp = {v[11]:f} at iteration {k}")
    if status == 5:
        raise InteriorViolationError("slacks and multipliers must be strictly positive and finite")
    if status == 4:
        if k == 0:
            raise NumericalBreakdownError(f"preconditioner produced r'P^{{-1}}r = {v[11]:f}")
        raise NumericalBreakdownError(f"r'P^{{-1}}r = {v[11]:f} at iteration {k}")
    res = PcgResult(ws.x, k, status == 1, float(v[10]), None)
    if not res.converged:
        raise NumericalBreakdownError(
            f"PCG stalled at preconditioned residual {res.residual_norm:.3e} "
            f"after {res.iterations} iterations")
    alpha_p, alpha_d = v[4], v[5]
    if min(alpha_p, alpha_d) < 1e-12:
        raise StalledError(
            f"fraction-to-boundary step collapsed (alpha_p={alpha_p:.2e}, alpha_d={alpha_d:.2e})")
    if v[7] != 0.0:
        raise StalledError("slack or multiplier left the strict interior")
    return res, alpha_p, alpha_d


def solve(b, mask: Mask, config: IpmConfig = IpmConfig(),
          observer=None) -> tuple[object, SolveReport]:
    """Run the interior-point method to the requested KKT tolerance (ipm.py:402-486).

    NumPy ``b`` -> NumPy ``beta`` (and NumPy state snapshots for the
    observer); a CUDA tensor ``b`` keeps everything on the device.
    """
    host = not _dev.is_device(b)
    if config.lam is not None and config.lam <= 0:
        raise ValueError("penalty must be positive")
    n = mask.shape.n
    # the 19 n-double workspace first; its PCG buffer then stages the upload
    # of host observations, so the peak is the workspace + b_hat (20 n)
    ws = Workspace(n)
    prob = Problem(b, mask, scratch=ws.work)
    lam = config.lam if config.lam is not None else prob.default_penalty(ws.g)
    if lam <= 0:
        raise ValueError("penalty must be positive")
    st = ws.state
    st.mu = lam / 2.0 if config.mu_init is None else float(config.mu_init)
    _lib.call("fl_ipm_init", n, ctypes.byref(ws.fs), float(lam), _dev.stream())

    t0 = time.perf_counter()
    records: list[IterationRecord] = []
    ws.best_beta.copy_(st.beta)
    best_kkt = math.inf
    status = "max_iters"
    prob.residual_adjoint(st.beta, ws.g)
    a = prob.assess(st, ws.g, lam, st.mu, ws.fs)
    conv = _conv_report(a, n, config.tol, config.gamma_centrality)

    for iteration in range(1, config.max_iters + 1):
        if conv.converged:
            status = "converged"
            break
        if a.barrier_residual <= config.inner_slack * st.mu:
            st.mu = next_barrier(st.mu, config.tol, config)

        t_iter = time.perf_counter()
        if _ASYNC_STEP:
            _launch_step(prob, ws, st.mu, lam, config)
            prob.residual_adjoint(st.beta, ws.g)
            a = prob.assess(st, ws.g, lam, st.mu, ws.fs)
            res, alpha_p, alpha_d = _step_verdict(ws)
        else:
            res, alpha_p, alpha_d = _fused_step(prob, ws, st.mu, lam, config)
            prob.residual_adjoint(st.beta, ws.g)
            a = prob.assess(st, ws.g, lam, st.mu, ws.fs)
        conv = _conv_report(a, n, config.tol, config.gamma_centrality)
        record = IterationRecord(
            iteration=iteration,
            mu=st.mu,
            primal_inf=conv.primal,
            dual_inf=max(conv.dual_equality, conv.multiplier_gap, conv.stationarity),
            complementarity=conv.complementarity,
            kkt_max=conv.max_residual,
            krylov_iters=res.iterations,
            alpha_primal=alpha_p,
            alpha_dual=alpha_d,
            pcg_residual=res.residual_norm,
            centrality_ok=conv.centrality_ok,
            wall_time=time.perf_counter() - t_iter,
        )
        records.append(record)
        if conv.max_residual < best_kkt:
            best_kkt = conv.max_residual
            ws.best_beta.copy_(st.beta)
        if observer is not None:
            # a fresh state per call, as the reference passes (ipm.py:382-393):
            # the solver updates st in place
            observer(st.to_numpy() if host else
                     IpmState(mu=st.mu, **{f: getattr(st, f).clone() for f in FIELDS}), record)
    else:
        if conv.converged:
            status = "converged"

    beta = st.beta if status == "converged" else ws.best_beta
    report = SolveReport(
        status=status,
        iterations=len(records),
        lam=lam,
        tol=config.tol,
        records=records,
        final_objective=prob.objective(beta, lam, ws.g),
        final_kkt=conv.max_residual if status == "converged" else best_kkt,
        final_mu=st.mu,
        wall_time=time.perf_counter() - t0,
    )
    return _dev.out(beta, host), report
