"""Seeded synthetic inputs for the BASELINE.json configs (host side, NumPy).

These build the *inputs* of a solve -- a sparse packed spectrum, a missing-
sample mask and a noise vector -- deterministically from NumPy's
``default_rng``.  The observed samples ``b = observe(beta, mask) + noise`` are
formed by the caller with whichever ``observe`` it is testing (the GPU one in
the product, the reference/oracle one when recording golden fixtures), so the
recipes themselves never touch a transform.

Recipes follow SURVEY.md Appendix A (C1..C5) plus the reference's own
product-of-harmonics generator (``synthetic.py:32-63``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Instance:
    """One synthetic problem before observation.

    ``flags`` marks missing samples (True = missing) on the flat grid;
    ``noise`` has one entry per *observed* sample.
    """

    dims: tuple
    beta_true: np.ndarray
    flags: np.ndarray
    noise: np.ndarray
    lam: float | None


def bragg_flags(n_side: int, spacing: int = 16, radius: float = 5.3) -> np.ndarray:
    """Bragg-peak punch mask: voxel missing within ``radius`` of a lattice point.

    A voxel (i, j, k) is missing when the squared periodic distance to the
    nearest multiple of ``spacing`` along every axis is <= radius**2
    (about 15.1% of the grid for the defaults).
    """
    t = np.arange(n_side) % spacing
    d = np.minimum(t, spacing - t).astype(np.int64) ** 2
    r2 = radius * radius
    # separable sum of squared distances, evaluated slab by slab to bound memory
    out = np.empty((n_side, n_side, n_side), dtype=bool)
    djk = d[:, None] + d[None, :]
    for i in range(n_side):
        out[i] = (d[i] + djk) <= r2
    return out.reshape(-1)


def c1_1d(seed: int = 0, n: int = 4096, miss: float = 0.10, dens: float = 0.01,
          noise: float = 0.05) -> Instance:
    """C1: 1D, 10% Bernoulli missing, 1% spikes, sigma=0.05, lambda=0.3."""
    rng = np.random.default_rng(seed)
    flags = rng.random(n) < miss
    beta = np.zeros(n)
    k = int(round(dens * n))
    idx = rng.choice(n, k, replace=False)
    beta[idx] = rng.uniform(1.0, 2.0, k) * rng.choice([-1.0, 1.0], k)
    n_obs = int(n - flags.sum())
    return Instance((n,), beta, flags, noise * rng.standard_normal(n_obs), 0.3)


def c2_2d(seed: int = 0, n_side: int = 2048, miss_target: float = 0.15,
          block=(8, 32), dens: float = 1e-4, noise: float = 0.05) -> Instance:
    """C2: 2D block-punched (~15% missing), sparse spectrum, default lambda."""
    rng = np.random.default_rng(seed)
    flags = np.zeros((n_side, n_side), bool)
    while flags.mean() < miss_target:
        s = rng.integers(block[0], block[1] + 1)
        i, j = rng.integers(0, n_side - s, 2)
        flags[i:i + s, j:j + s] = True
    n = n_side * n_side
    beta = np.zeros(n)
    k = max(1, int(round(dens * n)))
    idx = rng.choice(n, k, replace=False)
    beta[idx] = rng.uniform(1.0, 2.0, k) * rng.choice([-1.0, 1.0], k) * np.sqrt(n) / 64
    flags = flags.reshape(-1)
    n_obs = int(n - flags.sum())
    return Instance((n_side, n_side), beta, flags, noise * rng.standard_normal(n_obs), None)


def c3_bragg(n_side: int, seed: int = 0, noise: float = 0.05) -> Instance:
    """C3: 3D Bragg-punched, scaled amplitudes, default lambda."""
    rng = np.random.default_rng(seed)
    flags = bragg_flags(n_side)
    n = n_side ** 3
    nnz = max(8, n // 10000)
    beta = np.zeros(n)
    idx = rng.choice(n, nnz, replace=False)
    beta[idx] = rng.uniform(1, 2, nnz) * rng.choice([-1., 1.], nnz) * np.sqrt(n) / 64
    n_obs = int(n - flags.sum())
    return Instance((n_side,) * 3, beta, flags, noise * rng.standard_normal(n_obs), None)


def c4_const(n_side: int) -> Instance:
    """C4/C5: 3D Bragg-punched, unit-scale amplitudes, lambda = 0.5 fixed."""
    rng = np.random.default_rng(1234)
    flags = bragg_flags(n_side)
    n = n_side ** 3
    nnz = max(8, n // 10000)
    beta = np.zeros(n)
    idx = rng.choice(n, nnz, replace=False)
    beta[idx] = rng.uniform(1, 2, nnz) * rng.choice([-1., 1.], nnz)
    n_obs = int(n - flags.sum())
    return Instance((n_side,) * 3, beta, flags, 0.05 * rng.standard_normal(n_obs), 0.5)


C4_SEED = 1234
C4_SIGMA = 0.05


def c4_spikes(n: int):
    """The C4/C5 recipe's sparse spectrum: global flat indices and values
    (c4_const's own host RNG stream, only n/10^4 positions)."""
    rng = np.random.default_rng(C4_SEED)
    nnz = max(8, n // 10000)
    idx = rng.choice(n, nnz, replace=False)
    val = rng.uniform(1, 2, nnz) * rng.choice([-1., 1.], nnz)
    return idx, val


def noisy_embed_device(x, bits, ext, off, stride, noise_seed: int, sigma: float = C4_SIGMA):
    """In place: x = Z (x + sigma * noise), noise drawn per GLOBAL voxel index
    (``fl_noisy_embed``), so a full grid and any slab decomposition of it get
    bitwise the same draws."""
    import ctypes

    from . import _dev, _lib

    arr = lambda v: (ctypes.c_int64 * 3)(*[int(t) for t in v])  # noqa: E731
    _lib.call("fl_noisy_embed", arr(ext), arr(off), arr(stride), int(noise_seed) & (2 ** 64 - 1), float(sigma),
              _dev.ptr(bits), _dev.ptr(x), _dev.stream())


def c4_const_device(n_side: int, noise_seed: int = 0):
    """C4/C5 recipe generated on the GPU -> (mask, b, beta_idx, beta_val, lam).

    The Bragg mask is built on the device (``masking.BraggMask``, bit-equal
    to ``bragg_flags``); the spikes are c4_const's own (``c4_spikes``); the
    observation noise is drawn on the device per global voxel index
    (``fl_noisy_embed``), so ``b`` is NOT NumPy-identical to c4_const, but it
    IS identical to the slab-sharded recipe (``sharded.c4_problem_device``)
    -- a C5-scale input without any n-sized host array.
    """
    import torch

    from . import _dev
    from .fourier import GridShape, synthesize
    from .masking import BraggMask, restrict

    shape = GridShape((n_side,) * 3)
    n = shape.n
    idx, val = c4_spikes(n)
    mask = BraggMask(shape)
    beta = torch.zeros(n, dtype=torch.float64, device=_dev.device())
    beta[torch.from_numpy(idx).to(beta.device)] = torch.from_numpy(val).to(beta.device)
    x = synthesize(beta, shape)
    del beta
    d = n_side
    noisy_embed_device(x, mask.on_device().bits, (d, d, d), (0, 0, 0), (d * d, d, 1), noise_seed)
    b = restrict(x, mask)
    del x
    return mask, b, idx, val, 0.5


def harmonics(dims, noise_seed: int = 0, missing_fraction: float = 0.15,
              missing_seed: int = 1):
    """Reference generator (synthetic.py:32-63): product-of-harmonics truth.

    Returns ``(noisy, flags, truth)`` on the full grid; the observed samples
    are ``noisy[~flags]``.
    """
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    x = np.ones(dims)
    for axis, (extent, mult) in enumerate(zip(dims, (1, 2, 3))):
        t = np.arange(extent)
        phase = 2.0 * np.pi * mult * t / extent
        shape = [1] * len(dims)
        shape[axis] = extent
        x = x * (np.cos(phase) + 2.0 * np.sin(phase)).reshape(shape)
    truth = x.reshape(-1)
    noisy = truth + np.random.default_rng(noise_seed).random(n)
    mrng = np.random.default_rng(missing_seed)
    while True:
        flags = mrng.random(n) < missing_fraction
        if not flags.all():
            break
    return noisy, flags, truth
