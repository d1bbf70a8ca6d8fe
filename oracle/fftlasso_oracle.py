"""CPU oracle for the fftlasso hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it.  The product package
``paper_2502_04217_b200`` never imports anything under ``oracle/`` and fails
loudly when its CUDA library is missing.

What it is
----------
A NumPy/SciPy restatement of the reference package ``fftlasso``
(``/root/reference/pkg/src/fftlasso``) for the matrix-free IPM path:
per-axis packed real transforms, masked observation operators, the condensed
KKT algebra, PCG and the interior-point driver.  Every function cites the
reference ``file:line`` it restates.  Elementwise formulas keep the
reference's exact left-to-right evaluation order, so on equal inputs they are
bitwise identical to the reference.

Third-party arithmetic: the reference's real FFTs are SciPy's pocketfft
(``scipy.fft.irfft``/``rfft`` with ``norm="ortho"``, reference
``fourier.py:182`` and ``fourier.py:190``); pinned only as ``scipy>=1.10``
(``pyproject.toml:10-13``).  This oracle calls the same functions (scipy
1.18.1, numpy 2.3.5 in this image).  The packing it wraps around them is the
published algorithm of ``fourier.py:172-198``.

Parity pinning
--------------
``oracle/make_golden.py`` imports the real reference (available only in the
build container) and writes ``tests/golden/*.npz``; the CPU test
``tests/test_oracle_golden.py`` checks this oracle against every fixture
(bitwise where the reference is deterministic, 1e-15 otherwise).  The
independent trig-formula matrix ``dense_synthesis`` (reference
``diagnostics.py:57-83``) pins the transform without any FFT code.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.fft

ROOT2 = math.sqrt(2.0)
PCG_ITER_CAP = 5000  # pcg.py:19


def _workers() -> int:
    # fourier.py:44-49 -- FFTLASSO_THREADS caps pocketfft's worker count
    cap = os.environ.get("FFTLASSO_THREADS")
    return max(1, int(cap)) if cap is not None else (os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# grid + transform (fourier.py)
# ---------------------------------------------------------------------------

def check_dims(dims) -> tuple[int, ...]:
    """fourier.py:65-73: 1..3 axes, each even and >= 2."""
    dims = tuple(int(d) for d in dims)
    if not 1 <= len(dims) <= 3:
        raise ValueError(f"need 1 to 3 axes, got {len(dims)}")
    if any(d < 2 or d % 2 for d in dims):
        raise ValueError(f"every axis must be even and >= 2, got {dims}")
    return dims


def _to_half_spectrum(packed_last: np.ndarray) -> np.ndarray:
    """fourier.py:176-181: packed fibre (last axis) -> rfft half spectrum."""
    m = packed_last.shape[-1]
    h = m // 2
    half = np.zeros(packed_last.shape[:-1] + (h + 1,), dtype=np.complex128)
    half[..., 0] = packed_last[..., 0]
    half[..., h] = packed_last[..., 1]
    if h > 1:
        half[..., 1:h] = (packed_last[..., 2:h + 1] + 1j * packed_last[..., h + 1:]) / ROOT2
    return half


def _from_half_spectrum(half: np.ndarray, m: int) -> np.ndarray:
    """fourier.py:191-197: rfft half spectrum -> packed fibre (last axis)."""
    h = m // 2
    out = np.empty(half.shape[:-1] + (m,), dtype=np.float64)
    out[..., 0] = half[..., 0].real
    out[..., 1] = half[..., h].real
    if h > 1:
        out[..., 2:h + 1] = ROOT2 * half[..., 1:h].real
        out[..., h + 1:] = ROOT2 * half[..., 1:h].imag
    return out


def synth_axis(grid: np.ndarray, axis: int) -> np.ndarray:
    """fourier.py:172-183 -- packed coefficients -> samples along ``axis``."""
    moved = np.moveaxis(grid, axis, -1)
    m = moved.shape[-1]
    x = scipy.fft.irfft(_to_half_spectrum(moved), n=m, axis=-1, norm="ortho",
                        workers=_workers())
    return np.moveaxis(x, -1, axis)


def analyze_axis(grid: np.ndarray, axis: int) -> np.ndarray:
    """fourier.py:186-198 -- samples -> packed coefficients along ``axis``."""
    moved = np.moveaxis(grid, axis, -1)
    m = moved.shape[-1]
    half = scipy.fft.rfft(moved, axis=-1, norm="ortho", workers=_workers())
    return np.moveaxis(_from_half_spectrum(half, m), -1, axis)


def synthesize(beta, dims) -> np.ndarray:
    """fourier.py:201-222 -- A beta, axes ascending, row-major flat output."""
    dims = check_dims(dims)
    x = np.asarray(beta, dtype=np.float64).reshape(dims)
    for ax in range(len(dims)):
        x = synth_axis(x, ax)
    return np.ascontiguousarray(x).reshape(-1)


def analyze(x, dims) -> np.ndarray:
    """fourier.py:225-235 -- A^T x, axes ascending."""
    dims = check_dims(dims)
    b = np.asarray(x, dtype=np.float64).reshape(dims)
    for ax in range(len(dims)):
        b = analyze_axis(b, ax)
    return np.ascontiguousarray(b).reshape(-1)


def dense_synthesis(dims) -> np.ndarray:
    """diagnostics.py:57-83 -- trig-formula synthesis matrix (no FFT code)."""
    def one_axis(m):
        t = np.arange(m)[:, None]
        a = np.zeros((m, m))
        a[:, 0] = 1.0
        a[:, 1] = (-1.0) ** np.arange(m)
        k = np.arange(1, m // 2)[None, :]
        if k.size:
            ang = 2.0 * np.pi * k * t / m
            a[:, 2:m // 2 + 1] = ROOT2 * np.cos(ang)
            a[:, m // 2 + 1:] = -ROOT2 * np.sin(ang)
        return a / math.sqrt(m)

    dims = check_dims(dims)
    a = one_axis(dims[0])
    for m in dims[1:]:
        a = np.kron(a, one_axis(m))
    return a


# ---------------------------------------------------------------------------
# masked observation operators (masking.py)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class OMask:
    """masking.py:22-51 -- sorted missing indices + boolean flags."""
    dims: tuple[int, ...]
    missing: np.ndarray
    missing_bool: np.ndarray

    @property
    def n(self) -> int:
        return int(np.prod(self.dims))

    @property
    def n_observed(self) -> int:
        return self.n - int(self.missing.size)


def make_mask(dims, missing=None, flags=None) -> OMask:
    """masking.py:39-51 (validation) and :61-69 (from_bool)."""
    dims = check_dims(dims)
    n = int(np.prod(dims))
    if flags is not None:
        flags = np.asarray(flags).reshape(-1).astype(bool)
        if flags.size != n:
            raise ValueError("mask size mismatch")
        missing = np.flatnonzero(flags)
    idx = np.asarray(missing if missing is not None else [], dtype=np.int64).reshape(-1)
    if idx.size and (idx[0] < 0 or idx[-1] >= n or np.any(np.diff(idx) <= 0)):
        raise ValueError("missing indices must be in range and strictly increasing")
    if idx.size >= n:
        raise ValueError("cannot mask every sample")
    fl = np.zeros(n, dtype=bool)
    fl[idx] = True
    return OMask(dims, idx, fl)


def observe(beta, mask: OMask) -> np.ndarray:
    """masking.py:81-87."""
    x = synthesize(beta, mask.dims)
    return x if mask.missing.size == 0 else x[~mask.missing_bool]


def embed(values, mask: OMask) -> np.ndarray:
    """masking.py:90-99."""
    full = np.zeros(mask.n)
    full[~mask.missing_bool] = np.asarray(values, dtype=np.float64).reshape(-1)
    return full


def observe_adjoint(values, mask: OMask) -> np.ndarray:
    """masking.py:102-104."""
    return analyze(embed(values, mask), mask.dims)


def gram(beta, mask: OMask) -> np.ndarray:
    """masking.py:107-118 -- synthesize, zero the missing samples, analyze."""
    x = synthesize(beta, mask.dims)
    if mask.missing.size:
        x[mask.missing] = 0.0
    return analyze(x, mask.dims)


# ---------------------------------------------------------------------------
# condensed KKT algebra (newton_system.py)
# ---------------------------------------------------------------------------

@dataclass
class OState:
    """ipm.py:85-110 -- primal-dual iterate."""
    beta: np.ndarray
    z: np.ndarray
    s1: np.ndarray
    s2: np.ndarray
    y1: np.ndarray
    y2: np.ndarray
    nu1: np.ndarray
    nu2: np.ndarray
    mu: float

    def duality_measure(self) -> float:
        # ipm.py:103-105
        return float(self.nu1 @ self.s1 + self.nu2 @ self.s2) / (2 * self.beta.size)

    def copy(self) -> "OState":
        return OState(*(getattr(self, f).copy() for f in
                        ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2")), mu=self.mu)


def diagonals(s1, s2, nu1, nu2):
    """newton_system.py:72-91 -> (sigma1, sigma2, lambda1, lambda2, D, B)."""
    for name, a in (("s1", s1), ("s2", s2), ("nu1", nu1), ("nu2", nu2)):
        a = np.asarray(a, dtype=np.float64)
        if a.size == 0 or np.any(a <= 0.0) or not np.all(np.isfinite(a)):
            raise ValueError(f"interior violation: {name}")
    sig1 = nu1 / s1
    sig2 = nu2 / s2
    lam1 = sig1 + sig2
    lam2 = sig1 - sig2
    dvec = sig1 + sig2 + 4.0 * sig1 * sig2
    bvec = dvec / (1.0 + lam1)
    return sig1, sig2, lam1, lam2, dvec, bvec


def newton_rhs(st: OState, b, mask: OMask, lam: float) -> dict:
    """newton_system.py:113-145 -- r1..r6 and the condensed (r_beta, r_c)."""
    sig1, sig2 = diagonals(st.s1, st.s2, st.nu1, st.nu2)[:2]
    r1 = observe_adjoint(b - observe(st.beta, mask), mask) + st.y1 - st.y2
    r2 = st.y1 + st.y2 - lam
    r3 = st.y1 - st.mu / st.s1
    r4 = st.y2 - st.mu / st.s2
    r5 = st.z + st.beta - st.s1
    r6 = st.z - st.beta - st.s2
    return dict(r1=r1, r2=r2, r3=r3, r4=r4, r5=r5, r6=r6,
                r_beta=r1 - r3 + r4 - sig1 * r5 + sig2 * r6,
                r_c=r2 - r3 - r4 - sig1 * r5 - sig2 * r6)


def kkt_apply(db, dz, diag, mask: OMask):
    """newton_system.py:148-152."""
    _, _, lam1, lam2, _, _ = diag
    return gram(db, mask) + lam1 * db + lam2 * dz, lam2 * db + lam1 * dz


def precond_apply(rb, rc, diag):
    """newton_system.py:155-159."""
    _, _, lam1, lam2, dvec, bvec = diag
    return (lam1 * rb - lam2 * rc) / dvec, -lam2 / dvec * rb + rc / bvec


def recover(db, dz, rhs: dict, diag):
    """newton_system.py:184-196 -> (d_s1, d_s2, d_y1, d_y2), condensed signs."""
    sig1, sig2 = diag[0], diag[1]
    dy1 = -sig1 * (db + dz + rhs["r5"]) - rhs["r3"]
    dy2 = sig2 * (db - dz - rhs["r6"]) - rhs["r4"]
    return (rhs["r3"] + dy1) / sig1, (rhs["r4"] + dy2) / sig2, dy1, dy2


# ---------------------------------------------------------------------------
# PCG (pcg.py)
# ---------------------------------------------------------------------------

@dataclass
class OPcg:
    solution: np.ndarray
    iterations: int
    converged: bool
    residual_norm: float
    history: list | None = None


def pcg(op, prec, rhs, abs_tol=1e-12, rel_tol=0.0, max_iters=None, history=False) -> OPcg:
    """pcg.py:57-127 -- PCG from x0 = 0, preconditioned-norm stopping test."""
    rhs = np.asarray(rhs, dtype=np.float64)
    limit = int(max_iters) if max_iters is not None else min(10 * rhs.size, PCG_ITER_CAP)
    x = np.zeros_like(rhs)
    r = rhs.copy()
    zv = prec(r)
    rho = float(r @ zv)
    if not math.isfinite(rho) or rho < 0:
        raise ArithmeticError(f"r'P^-1 r = {rho}")
    norm = math.sqrt(rho)
    thr = abs_tol + rel_tol * norm
    hist = [norm] if history else None
    if norm <= thr:
        return OPcg(x, 0, True, norm, hist)
    p = zv.copy()
    for k in range(1, limit + 1):
        kp = op(p)
        curv = float(p @ kp)
        if not math.isfinite(curv) or curv <= 0:
            raise ArithmeticError(f"curvature {curv} at iteration {k}")
        alpha = rho / curv
        x += alpha * p
        r -= alpha * kp
        zv = prec(r)
        rho_next = float(r @ zv)
        if not math.isfinite(rho_next) or rho_next < 0:
            raise ArithmeticError(f"r'P^-1 r = {rho_next} at iteration {k}")
        norm = math.sqrt(rho_next)
        if hist is not None:
            hist.append(norm)
        if norm <= thr:
            return OPcg(x, k, True, norm, hist)
        p = zv + (rho_next / rho) * p
        rho = rho_next
    return OPcg(x, limit, False, norm, hist)


# ---------------------------------------------------------------------------
# interior-point driver (ipm.py)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class OConfig:
    """ipm.py:55-82 defaults."""
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


def _maxabs(v) -> float:
    return float(np.max(np.abs(v))) if v.size else 0.0  # ipm.py:200-201


def default_penalty(b, mask: OMask) -> float:
    """ipm.py:204-206."""
    return 0.1 * float(np.max(np.abs(observe_adjoint(b, mask))))


def lasso_objective(beta, b, mask: OMask, lam: float) -> float:
    """ipm.py:209-211."""
    res = b - observe(beta, mask)
    return 0.5 * float(res @ res) + lam * float(np.sum(np.abs(beta)))


def initial_state(n: int, lam: float, mu_init=None) -> OState:
    """ipm.py:214-238."""
    if lam <= 0:
        raise ValueError("penalty must be positive")
    e = np.ones(n)
    half = 0.5 * lam * e
    return OState(np.zeros(n), e.copy(), e.copy(), e.copy(), half.copy(), half.copy(),
                  half.copy(), half.copy(), lam / 2.0 if mu_init is None else float(mu_init))


def kkt_check(st: OState, b, mask: OMask, lam: float, tol: float, gamma=1e-4) -> dict:
    """ipm.py:241-273 -- exact (mu = 0) KKT residual norms."""
    stat = observe_adjoint(b - observe(st.beta, mask), mask) + st.y1 - st.y2
    p1 = st.s1 * st.nu1
    p2 = st.s2 * st.nu2
    out = dict(
        stationarity=_maxabs(stat),
        dual_equality=_maxabs(lam - st.y1 - st.y2),
        multiplier_gap=max(_maxabs(st.y1 - st.nu1), _maxabs(st.y2 - st.nu2)),
        primal=max(_maxabs(st.z + st.beta - st.s1), _maxabs(st.z - st.beta - st.s2)),
        complementarity=max(float(p1.max()), float(p2.max())),
    )
    out["max_residual"] = max(out["stationarity"], out["dual_equality"],
                              out["multiplier_gap"], out["primal"], out["complementarity"])
    out["converged"] = out["max_residual"] <= tol
    out["duality_measure"] = st.duality_measure()
    out["centrality_ok"] = bool(min(p1.min(), p2.min()) >= gamma * out["duality_measure"])
    return out


def barrier_residual(st: OState, rhs: dict) -> float:
    """ipm.py:276-282."""
    pieces = [rhs["r1"], rhs["r2"], rhs["r5"], rhs["r6"], st.s1 * st.nu1 - st.mu,
              st.s2 * st.nu2 - st.mu, st.y1 - st.nu1, st.y2 - st.nu2]
    return max(float(np.max(np.abs(p))) for p in pieces)


def newton_direction(st: OState, b, mask: OMask, lam: float, cfg: OConfig) -> dict:
    """ipm.py:303-352 -- condensed PCG solve + back-substitution + sign flip."""
    n = st.beta.size
    diag = diagonals(st.s1, st.s2, st.nu1, st.nu2)
    rhs = newton_rhs(st, b, mask, lam)
    res = pcg(lambda v: np.concatenate(kkt_apply(v[:n], v[n:], diag, mask)),
              lambda v: np.concatenate(precond_apply(v[:n], v[n:], diag)),
              np.concatenate([rhs["r_beta"], rhs["r_c"]]),
              abs_tol=cfg.cg_tol, max_iters=cfg.cg_max_iters)
    if not res.converged:
        raise ArithmeticError(f"PCG stalled at {res.residual_norm:.3e}")
    db, dz = res.solution[:n], res.solution[n:]
    ds1, ds2, dy1, dy2 = recover(db, dz, rhs, diag)
    ds1 = -ds1
    ds2 = -ds2
    dnu1 = (st.mu - st.s1 * st.nu1) / st.s1 - diag[0] * ds1
    dnu2 = (st.mu - st.s2 * st.nu2) / st.s2 - diag[1] * ds2
    return dict(d_beta=db, d_z=dz, d_s1=ds1, d_s2=ds2, d_y1=dy1, d_y2=dy2,
                d_nu1=dnu1, d_nu2=dnu2, krylov_iters=res.iterations,
                pcg_residual=res.residual_norm)


def fraction_to_boundary(v, dv, tau: float) -> float:
    """ipm.py:355-361."""
    neg = dv < 0.0
    if not np.any(neg):
        return 1.0
    return min(1.0, tau * float(np.min(v[neg] / -dv[neg])))


def ipm_step(st: OState, b, mask: OMask, lam: float, cfg: OConfig):
    """ipm.py:364-394."""
    d = newton_direction(st, b, mask, lam, cfg)
    tau = max(cfg.ftb_tau, 1.0 - st.mu)
    ap = min(fraction_to_boundary(st.s1, d["d_s1"], tau),
             fraction_to_boundary(st.s2, d["d_s2"], tau))
    ad = min(fraction_to_boundary(st.nu1, d["d_nu1"], tau),
             fraction_to_boundary(st.nu2, d["d_nu2"], tau))
    if min(ap, ad) < 1e-12:
        raise RuntimeError(f"stalled: alpha_p={ap:.2e} alpha_d={ad:.2e}")
    new = OState(st.beta + ap * d["d_beta"], st.z + ap * d["d_z"],
                 st.s1 + ap * d["d_s1"], st.s2 + ap * d["d_s2"],
                 st.y1 + ad * d["d_y1"], st.y2 + ad * d["d_y2"],
                 st.nu1 + ad * d["d_nu1"], st.nu2 + ad * d["d_nu2"], st.mu)
    for f in ("s1", "s2", "nu1", "nu2"):
        if np.any(getattr(new, f) <= 0.0):
            raise RuntimeError(f"stalled: {f} left the interior")
    return new, d, ap, ad


def next_barrier(mu: float, tol: float, cfg: OConfig) -> float:
    """ipm.py:397-399."""
    return max(tol / 10.0, min(cfg.sigma_mu * mu, mu ** cfg.mu_power))


@dataclass
class OReport:
    status: str
    iterations: int
    lam: float
    records: list = field(default_factory=list)
    final_objective: float = 0.0
    final_kkt: float = 0.0
    final_mu: float = 0.0
    wall_time: float = 0.0

    @property
    def krylov_counts(self) -> list:
        return [r["krylov_iters"] for r in self.records]


def solve(b, mask: OMask, cfg: OConfig = OConfig(), observer=None):
    """ipm.py:402-486 -- the outer loop with best-iterate return."""
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    lam = cfg.lam if cfg.lam is not None else default_penalty(b, mask)
    st = initial_state(mask.n, lam, cfg.mu_init)
    t0 = time.perf_counter()
    records = []
    best_beta, best_kkt = st.beta.copy(), math.inf
    status = "max_iters"
    conv = kkt_check(st, b, mask, lam, cfg.tol, cfg.gamma_centrality)
    for it in range(1, cfg.max_iters + 1):
        if conv["converged"]:
            status = "converged"
            break
        rhs = newton_rhs(st, b, mask, lam)
        if barrier_residual(st, rhs) <= cfg.inner_slack * st.mu:
            st.mu = next_barrier(st.mu, cfg.tol, cfg)
        t_it = time.perf_counter()
        st, d, ap, ad = ipm_step(st, b, mask, lam, cfg)
        conv = kkt_check(st, b, mask, lam, cfg.tol, cfg.gamma_centrality)
        rec = dict(record="iteration", iteration=it, mu=st.mu, primal_inf=conv["primal"],
                   dual_inf=max(conv["dual_equality"], conv["multiplier_gap"],
                                conv["stationarity"]),
                   complementarity=conv["complementarity"], kkt_max=conv["max_residual"],
                   krylov_iters=d["krylov_iters"], alpha_primal=ap, alpha_dual=ad,
                   pcg_residual=d["pcg_residual"], centrality_ok=conv["centrality_ok"],
                   wall_time=time.perf_counter() - t_it)
        records.append(rec)
        if conv["max_residual"] < best_kkt:
            best_kkt = conv["max_residual"]
            best_beta = st.beta.copy()
        if observer is not None:
            observer(st, rec)
    else:
        if conv["converged"]:
            status = "converged"
    beta = st.beta if status == "converged" else best_beta
    rep = OReport(status, len(records), lam, records,
                  final_objective=lasso_objective(beta, b, mask, lam),
                  final_kkt=conv["max_residual"] if status == "converged" else best_kkt,
                  final_mu=st.mu, wall_time=time.perf_counter() - t0)
    return beta, rep


# ---------------------------------------------------------------------------
# diagnostics.py: soft threshold, support classification, ISTA cross-check
# ---------------------------------------------------------------------------

def soft_threshold(x, t: float) -> np.ndarray:
    """diagnostics.py:325-328: sign(x) * max(|x| - t, 0)."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.maximum(np.abs(x) - t, 0.0)


def support(beta, threshold=None):
    """diagnostics.py:129-142 -> (positive, negative, zero, threshold)."""
    beta = np.asarray(beta, dtype=np.float64).reshape(-1)
    if threshold is None:
        threshold = 1e-6 * (float(np.max(np.abs(beta))) if beta.size else 0.0)
    return (np.flatnonzero(beta > threshold), np.flatnonzero(beta < -threshold),
            np.flatnonzero(np.abs(beta) <= threshold), float(threshold))


def dense_gram(mask: OMask) -> np.ndarray:
    """diagnostics.py:86-91 -- M_perp^T M_perp from the trig-formula matrix."""
    a = dense_synthesis(mask.dims)[~mask.missing_bool, :]
    return a.T @ a


def dense_condensed(st, mask: OMask):
    """diagnostics.py:94-108 -- dense (K, P) of the condensed system at an iterate."""
    _, _, lam1, lam2, _, _ = diagonals(st.s1, st.s2, st.nu1, st.nu2)
    g = dense_gram(mask)
    k = np.block([[g + np.diag(lam1), np.diag(lam2)], [np.diag(lam2), np.diag(lam1)]])
    p = np.block([[np.diag(1.0 + lam1), np.diag(lam2)], [np.diag(lam2), np.diag(lam1)]])
    return k, p


def dense_augmented(st, mask: OMask) -> np.ndarray:
    """Reference tests/conftest.py:20-39 -- the 6n x 6n symmetrised Newton
    matrix in the order (d_beta, d_z, d_s1, d_s2, d_y1, d_y2)."""
    n = np.asarray(st.beta).size
    g = dense_gram(mask)
    i, z = np.eye(n), np.zeros((n, n))
    sg1, sg2 = np.diag(st.nu1 / st.s1), np.diag(st.nu2 / st.s2)
    return np.block([[g, z, z, z, -i, i], [z, z, z, z, -i, -i], [z, z, sg1, z, -i, z],
                     [z, z, z, sg2, z, -i], [-i, -i, -i, z, z, z], [i, -i, z, -i, z, z]])


def preconditioned_spectrum(st, mask: OMask, cluster_tol: float = 0.05, support_threshold=None) -> dict:
    """diagnostics.py:183-224 -- dense eigen-probe of P^-1 K (as K v = l P v)."""
    import scipy.linalg

    n = np.asarray(st.beta).size
    if n > 1024:
        raise ValueError(f"spectrum probe guard: n {n} > 1024")
    k, p = dense_condensed(st, mask)
    eigs = scipy.linalg.eigh(k, p, eigvals_only=True)
    eigs_k = scipy.linalg.eigvalsh(k)
    pos, neg, _, _ = support(st.beta, support_threshold)
    active = np.sort(np.concatenate([pos, neg]))
    if active.size:
        q_eigs = scipy.linalg.eigvalsh(dense_gram(mask)[np.ix_(active, active)])
        kappa_pred = max(1.0, float(q_eigs[-1])) / min(1.0, float(q_eigs[0]))
    else:
        kappa_pred = 1.0
    comp_floor = min(float(np.min(st.s1 + st.nu1)), float(np.min(st.s2 + st.nu2)))
    return dict(eigenvalues=eigs, unit_cluster_size=int(np.sum(np.abs(eigs - 1.0) <= cluster_tol)),
                predicted_cluster_size=2 * n - int(active.size),
                kappa_observed=float(eigs[-1] / eigs[0]), kappa_predicted=kappa_pred,
                kappa_unpreconditioned=float(eigs_k[-1] / eigs_k[0]), n_active=int(active.size),
                strict_complementarity=comp_floor,
                duality_measure=(float(np.dot(st.nu1, st.s1)) + float(np.dot(st.nu2, st.s2))) / (2 * n))


def ista(b, mask: OMask, lam: float, tol: float = 1e-10, max_iters: int = 10**6):
    """diagnostics.py:331-360 without the n <= 4096 guard -> (beta, iterations).

    Unit-step proximal gradient: grad = G beta - xi, beta+ = soft(beta - grad,
    lam), stop when max|beta+ - beta| <= tol; raises RuntimeError at the cap
    (the reference raises IterationLimitError, a RuntimeError).
    """
    xi = observe_adjoint(np.asarray(b, dtype=np.float64).reshape(-1), mask)
    beta = np.zeros(mask.n)
    for k in range(1, max_iters + 1):
        nxt = soft_threshold(beta - (gram(beta, mask) - xi), lam)
        step = float(np.max(np.abs(nxt - beta))) if beta.size else 0.0
        beta = nxt
        if step <= tol:
            return beta, k
    raise RuntimeError(f"ISTA did not reach tol={tol:.1e} within {max_iters} iterations")
