"""Masked observation operators, B200 path (reference masking.py).

``Mask`` keeps the reference's host representation (sorted int64 indices +
boolean flags, masking.py:22-69) and lazily builds, per device, the bitmask
the kernels test (n/8 bytes) plus per-32-voxel observed-count offsets for
the gather/scatter kernels.  ``gram`` is one fused multi-pass operator
(2d-1 HBM passes, csrc/fl_pass.cu); ``observe`` / ``observe_adjoint`` are a
transform plus a bitmask gather / scatter kernel.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from .errors import UnsupportedShapeError
from .fourier import GridShape

__all__ = ["Mask", "BraggMask", "observe", "observe_adjoint", "gram", "embed", "restrict"]


class DeviceMask:
    """Bitmask + offsets of a Mask on one device."""

    def __init__(self, mask: "Mask"):
        import torch

        dev = _dev.device()
        n = mask.shape.n
        nw = (n + 31) // 32
        flags = torch.from_numpy(mask.missing_bool.view(np.uint8)).to(dev)
        self.bits = torch.empty(nw, dtype=torch.int32, device=dev)
        self.offsets = torch.empty(nw, dtype=torch.int64, device=dev)
        n_obs = ctypes.c_int64()
        _lib.call("fl_mask_build", n, _dev.ptr(flags), _dev.ptr(self.bits), _dev.ptr(self.offsets),
                  ctypes.byref(n_obs), _dev.stream())
        if n_obs.value != mask.n_observed:
            raise RuntimeError("device mask disagrees with host mask")
        self.n_observed = n_obs.value
        self.device = dev


@dataclass(frozen=True)
class Mask:
    """Missing-sample index set on a grid (masking.py:22-69)."""

    missing: np.ndarray
    shape: GridShape
    missing_bool: np.ndarray = field(init=False, repr=False, compare=False)
    _dev_cache: dict = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        idx = np.asarray(self.missing, dtype=np.int64).reshape(-1)
        if idx.size:
            if idx[0] < 0 or idx[-1] >= self.shape.n:
                raise ValueError("missing indices out of range")
            if np.any(np.diff(idx) <= 0):
                raise ValueError("missing indices must be strictly increasing")
        if idx.size >= self.shape.n:
            raise ValueError("cannot mask every sample")
        flags = np.zeros(self.shape.n, dtype=bool)
        flags[idx] = True
        object.__setattr__(self, "missing", idx)
        object.__setattr__(self, "missing_bool", flags)
        object.__setattr__(self, "_dev_cache", {})

    @property
    def n_missing(self) -> int:
        return int(self.missing.size)

    @property
    def n_observed(self) -> int:
        return self.shape.n - self.n_missing

    @classmethod
    def from_bool(cls, flags, shape: GridShape) -> "Mask":
        flags = np.asarray(flags).reshape(-1).astype(bool)
        if flags.size != shape.n:
            raise UnsupportedShapeError(f"mask has {flags.size} entries, grid expects {shape.n}")
        return cls(np.flatnonzero(flags), shape)

    def on_device(self) -> DeviceMask:
        dev = _dev.device()
        dm = self._dev_cache.get(dev.index)
        if dm is None:
            dm = DeviceMask(self)
            self._dev_cache[dev.index] = dm
        return dm


class BraggMask:
    """The Bragg-peak punch mask of the C3-C5 recipes, generated on the GPU.

    Same missing set as ``Mask.from_bool(workloads.bragg_flags(...), shape)``
    (bit for bit), built straight into the device bitmask and observed
    offsets (``fl_mask_bragg``) -- no n-byte host flags, no index array, so a
    C5-sized problem needs no host-side mask at all.
    Usable wherever the solver takes a ``Mask``; ``missing`` /
    ``missing_bool`` are materialised on the host only if asked for.
    """

    def __init__(self, shape: GridShape, spacing: int = 16, radius: float = 5.3):
        import torch

        self.shape = shape
        dev = _dev.device()
        nw = (shape.n + 31) // 32
        bits = torch.empty(nw, dtype=torch.int32, device=dev)
        offsets = torch.empty(nw, dtype=torch.int64, device=dev)
        dims = (ctypes.c_int64 * shape.ndim)(*shape.dims)
        n_obs = ctypes.c_int64()
        _lib.call("fl_mask_bragg", shape.ndim, dims, int(spacing), float(radius), _dev.ptr(bits),
                  _dev.ptr(offsets), ctypes.byref(n_obs), _dev.stream())
        if n_obs.value <= 0:
            raise ValueError("cannot mask every sample")
        dm = DeviceMask.__new__(DeviceMask)
        dm.bits, dm.offsets, dm.n_observed, dm.device = bits, offsets, n_obs.value, dev
        self._dm = dm
        self._host = None

    @property
    def n_observed(self) -> int:
        return self._dm.n_observed

    @property
    def n_missing(self) -> int:
        return self.shape.n - self._dm.n_observed

    def on_device(self) -> DeviceMask:
        if _dev.device() != self._dm.device:
            raise ValueError("BraggMask lives on the device it was built on")
        return self._dm

    @property
    def missing_bool(self) -> np.ndarray:
        if self._host is None:
            words = self._dm.bits.cpu().numpy().view(np.uint32)
            flags = np.unpackbits(words.view(np.uint8), bitorder="little")[: self.shape.n].astype(bool)
            self._host = flags
        return self._host

    @property
    def missing(self) -> np.ndarray:
        return np.flatnonzero(self.missing_bool)


def _coeffs(beta, mask: Mask):
    return _dev.to_dev(beta, mask.shape.n, "coefficient vector")


def embed_device(values_dev, mask: Mask):
    """embed on device tensors (no size check beyond n_observed)."""
    dm = mask.on_device()
    full = _dev.empty(mask.shape.n)
    _lib.call("fl_embed", mask.shape.n, _dev.ptr(dm.bits), _dev.ptr(dm.offsets),
              _dev.ptr(values_dev), _dev.ptr(full), _dev.stream())
    return full


def observe(beta, mask: Mask):
    """Synthesize and keep the observed samples in index order (masking.py:81-87)."""
    host = not _dev.is_device(beta)
    src = _coeffs(beta, mask)
    plan = _dev.plan_for(mask.shape.dims)
    x = _dev.empty(mask.shape.n)
    _lib.call("fl_synthesize", plan.handle, _dev.ptr(src), _dev.ptr(x), _dev.stream())
    if mask.n_missing == 0:
        return _dev.out(x, host)
    dm = mask.on_device()
    obs = _dev.empty(mask.n_observed)
    _lib.call("fl_gather_observed", mask.shape.n, _dev.ptr(dm.bits), _dev.ptr(dm.offsets),
              _dev.ptr(x), _dev.ptr(obs), _dev.stream())
    return _dev.out(obs, host)


def restrict(values, mask: Mask):
    """values[~mask.missing_bool] for a full-grid volume, gathered on the device.

    The CLI's ``b = values[~mask.missing_bool]`` (cli.py:73) without a host
    pass; NumPy in -> NumPy out, CUDA tensor in -> CUDA tensor out.
    """
    host = not _dev.is_device(values)
    v = _dev.to_dev(values, mask.shape.n, "volume")
    if mask.n_missing == 0:
        return _dev.out(v.clone(), host)
    dm = mask.on_device()
    obs = _dev.empty(mask.n_observed)
    _lib.call("fl_gather_observed", mask.shape.n, _dev.ptr(dm.bits), _dev.ptr(dm.offsets),
              _dev.ptr(v), _dev.ptr(obs), _dev.stream())
    return _dev.out(obs, host)


def embed(values, mask: Mask):
    """Zero-fill observed values back onto the full grid (masking.py:90-99)."""
    host = not _dev.is_device(values)
    v = _dev.to_dev(values, None)
    if v.numel() != mask.n_observed:
        raise UnsupportedShapeError(
            f"observed vector has {v.numel()} entries, mask expects {mask.n_observed}")
    return _dev.out(embed_device(v, mask), host)


def observe_adjoint(values, mask: Mask):
    """Zero-fill, then analyze (masking.py:102-104)."""
    host = not _dev.is_device(values)
    v = _dev.to_dev(values, None)
    if v.numel() != mask.n_observed:
        raise UnsupportedShapeError(
            f"observed vector has {v.numel()} entries, mask expects {mask.n_observed}")
    full = embed_device(v, mask)
    plan = _dev.plan_for(mask.shape.dims)
    _lib.call("fl_analyze", plan.handle, _dev.ptr(full), _dev.ptr(full), _dev.stream())
    return _dev.out(full, host)


def gram(beta, mask: Mask):
    """M^T M beta on the full grid in one fused operator (masking.py:107-118)."""
    host = not _dev.is_device(beta)
    src = _coeffs(beta, mask)
    plan = _dev.plan_for(mask.shape.dims)
    dm = mask.on_device()
    dst = _dev.empty(mask.shape.n)
    _lib.call("fl_gram", plan.handle, _dev.ptr(dm.bits), _dev.ptr(src), _dev.ptr(dst), _dev.stream())
    return _dev.out(dst, host)
