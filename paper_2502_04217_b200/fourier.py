"""Orthogonal real-packing Fourier transform, B200 path (reference fourier.py).

``synthesize`` (A) and ``analyze`` (A^T) run as fp64 CUDA passes of
libfftlasso_b200 (csrc/fl_pass.cu): one HBM pass per axis, fibres paired
into complex FFTs, packing and the ortho scale fused into the load/store
stages.  ``pack``/``unpack`` convert between a conjugate-symmetric complex
spectrum and packed coefficients; they are host-side API conveniences that
are not on the solver path (reference fourier.py:126-169).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from .errors import MalformedSpectrumError, UnsupportedShapeError

__all__ = ["GridShape", "pack", "unpack", "synthesize", "analyze"]

SYMMETRY_RTOL = 1e-10  # fourier.py:39
_SQRT2 = math.sqrt(2.0)


def _fft_workers() -> int:
    """API parity with fourier.py:44-49 (FFTLASSO_THREADS cap).  The GPU path
    has no host FFT workers; the value is reported, not used."""
    cap = os.environ.get("FFTLASSO_THREADS")
    if cap is not None:
        return max(1, int(cap))
    return os.cpu_count() or 1


@dataclass(frozen=True)
class GridShape:
    """Grid geometry: 1 to 3 axes, every extent even and >= 2 (fourier.py:52-77)."""

    dims: tuple[int, ...]
    n: int = field(init=False)

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        if not 1 <= len(dims) <= 3:
            raise UnsupportedShapeError(f"need 1 to 3 axes, got {len(dims)}")
        for d in dims:
            if d < 2 or d % 2 != 0:
                raise UnsupportedShapeError(f"every axis must be even and >= 2, got {d}")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "n", int(np.prod(dims)))

    @property
    def ndim(self) -> int:
        return len(self.dims)


def _grid(values, shape: GridShape, dtype) -> np.ndarray:
    arr = np.asarray(values, dtype=dtype)
    if arr.size != shape.n:
        raise UnsupportedShapeError(f"array has {arr.size} elements, grid expects {shape.n}")
    return arr.reshape(shape.dims)


def _pack_fibres(v: np.ndarray) -> np.ndarray:
    """Unitary packing along the last axis of a complex array."""
    m = v.shape[-1]
    h = m // 2
    out = np.empty_like(v)
    out[..., 0] = v[..., 0]
    out[..., 1] = v[..., h]
    if h > 1:
        lo = v[..., 1:h]
        hi = v[..., m - 1:h:-1]  # v[m-k], k = 1..h-1
        out[..., 2:h + 1] = (lo + hi) / _SQRT2
        out[..., h + 1:] = 1j * (hi - lo) / _SQRT2
    return out


def _unpack_fibres(b: np.ndarray) -> np.ndarray:
    """Adjoint of :func:`_pack_fibres` along the last axis."""
    m = b.shape[-1]
    h = m // 2
    out = np.empty_like(b)
    out[..., 0] = b[..., 0]
    out[..., h] = b[..., 1]
    if h > 1:
        re = b[..., 2:h + 1]
        im = b[..., h + 1:]
        out[..., 1:h] = (re + 1j * im) / _SQRT2
        out[..., m - 1:h:-1] = (re - 1j * im) / _SQRT2
    return out


def _per_axis(w: np.ndarray, fn) -> np.ndarray:
    for axis in range(w.ndim):
        w = np.moveaxis(fn(np.moveaxis(w, axis, -1)), -1, axis)
    return w


def pack(v, shape: GridShape) -> np.ndarray:
    """Conjugate-symmetric spectrum -> real packed coefficients (fourier.py:126-157)."""
    w = _grid(v, shape, np.complex128)
    scale = float(np.max(np.abs(w))) if w.size else 0.0
    w = _per_axis(w, _pack_fibres)
    residue = float(np.max(np.abs(w.imag))) if w.size else 0.0
    if residue > SYMMETRY_RTOL * max(scale, 1e-300):
        raise MalformedSpectrumError(
            f"spectrum is not conjugate-symmetric: residue {residue:.3e} "
            f"exceeds {SYMMETRY_RTOL:.0e} * {scale:.3e}")
    return np.ascontiguousarray(w.real).reshape(-1)


def unpack(beta, shape: GridShape) -> np.ndarray:
    """Packed coefficients -> full conjugate-symmetric spectrum (fourier.py:160-169)."""
    w = _grid(beta, shape, np.float64).astype(np.complex128)
    return _per_axis(w, _unpack_fibres).reshape(-1)


def synthesize(beta, shape: GridShape):
    """A beta on the GPU (fourier.py:201-222).  NumPy in -> NumPy out."""
    host = not _dev.is_device(beta)
    src = _dev.to_dev(beta, shape.n, "coefficient vector")
    plan = _dev.plan_for(shape.dims)
    dst = _dev.empty(shape.n)
    _lib.call("fl_synthesize", plan.handle, _dev.ptr(src), _dev.ptr(dst), _dev.stream())
    return _dev.out(dst, host)


def analyze(x, shape: GridShape):
    """A^T x on the GPU (fourier.py:225-235).  NumPy in -> NumPy out."""
    host = not _dev.is_device(x)
    src = _dev.to_dev(x, shape.n, "signal")
    plan = _dev.plan_for(shape.dims)
    dst = _dev.empty(shape.n)
    _lib.call("fl_analyze", plan.handle, _dev.ptr(src), _dev.ptr(dst), _dev.stream())
    return _dev.out(dst, host)
