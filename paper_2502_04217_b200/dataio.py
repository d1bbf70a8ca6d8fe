"""Volume and mask files, format-compatible with the reference (dataio.py:1-109).

On disk (unchanged, so files move freely between the two packages):

* volume  ``path``: raw little-endian float64 samples, row-major;
  ``path + ".json"``: ``{"dims": [...], "order": "row-major", "dtype": "f64-le"}``
* mask    ``path``: sorted uint64-le missing indices (``"indices"``) or one
  byte per grid sample, nonzero = missing (``"bytemask"``);
  ``path + ".json"``: ``{"format": ..., "dims": [...]}``

B200 specifics: payloads are read with one ``readinto`` straight into a
page-locked buffer from torch's caching host allocator when a CUDA device is
present, so the host->device copy that follows is a full-bandwidth DMA and
no second host copy is made; ``write_volume`` takes CUDA tensors too (one
device->host copy into pinned memory).  Header errors raise ``ValueError``
with the reference's wording.  File handling is host work and needs no GPU.
"""

from __future__ import annotations

import json
import os

import numpy as np

from .fourier import GridShape
from .masking import Mask

__all__ = ["read_volume", "write_volume", "read_mask", "write_mask", "sidecar_path"]

VOLUME_DTYPE = "f64-le"
VOLUME_ORDER = "row-major"
MASK_FORMATS = ("indices", "bytemask")


def sidecar_path(path: str) -> str:
    """Header file next to a payload (dataio.py:35-36)."""
    return path + ".json"


def _header(path: str) -> dict:
    """Parse and minimally validate a sidecar (dataio.py:39-50)."""
    side = sidecar_path(path)
    if not os.path.exists(side):
        raise ValueError(f"missing header sidecar {side}")
    try:
        with open(side, encoding="utf-8") as fh:
            meta = json.load(fh)
    except json.JSONDecodeError as exc:
        raise ValueError(f"malformed header {side}: {exc}") from exc
    if isinstance(meta, dict) and "dims" in meta:
        return meta
    raise ValueError(f"malformed header {side}: missing 'dims'")


def _put_header(path: str, meta: dict) -> None:
    with open(sidecar_path(path), "w", encoding="utf-8") as fh:
        fh.write(json.dumps(meta) + "\n")


def _staging(count: int, dtype) -> np.ndarray:
    """Host array for a payload: pinned (DMA-able) when CUDA is usable."""
    try:
        import torch
    except ImportError:  # pragma: no cover - torch is part of the image
        return np.empty(count, dtype=dtype)
    if not torch.cuda.is_available():
        return np.empty(count, dtype=dtype)
    t = torch.empty(count, dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True)
    return t.numpy()


def _slurp(path: str, dtype) -> np.ndarray:
    """Whole items of ``path`` as ``dtype`` (same truncation rule as np.fromfile)."""
    item = np.dtype(dtype).itemsize
    count = os.path.getsize(path) // item
    arr = _staging(count, dtype)
    if count:
        with open(path, "rb") as fh:
            if fh.readinto(arr.view(np.uint8)) != count * item:
                raise OSError(f"short read from {path}")
    return arr


def _host_f64(values, expected: int, dims) -> np.ndarray:
    """Flat little-endian float64 host view of NumPy data or a (CUDA) tensor."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(values, torch.Tensor):
        t = values.detach().reshape(-1)
        if t.is_cuda:
            host = torch.empty(t.numel(), dtype=torch.float64, pin_memory=True)
            host.copy_(t)
            values = host.numpy()
        else:
            values = t.to(torch.float64).numpy()
    flat = np.asarray(values, dtype="<f8").reshape(-1)
    if flat.size != expected:
        raise ValueError(f"payload has {flat.size} samples, dims {list(dims)} expect {expected}")
    return flat


def write_volume(path: str, values, dims) -> None:
    """Payload + sidecar (dataio.py:53-64); ``values`` may live on the GPU."""
    dims = [int(d) for d in dims]
    _host_f64(values, int(np.prod(dims)), dims).tofile(path)
    _put_header(path, {"dims": dims, "order": VOLUME_ORDER, "dtype": VOLUME_DTYPE})


def read_volume(path: str) -> tuple[np.ndarray, tuple[int, ...]]:
    """(flat float64 samples, dims) (dataio.py:67-82); pinned when CUDA is up."""
    meta = _header(path)
    dims = tuple(int(d) for d in meta["dims"])
    for key, want in (("dtype", VOLUME_DTYPE), ("order", VOLUME_ORDER)):
        got = meta.get(key, want)
        if got != want:
            raise ValueError(f"unsupported {key} {got!r} in {path}")
    samples = _slurp(path, np.dtype("<f8"))
    n = int(np.prod(dims))
    if samples.size != n:
        raise ValueError(f"volume {path} has {samples.size} samples, header dims {dims} expect {n}")
    return samples, dims


def write_mask(path: str, mask: Mask, fmt: str = "indices") -> None:
    """dataio.py:85-96."""
    if fmt not in MASK_FORMATS:
        raise ValueError(f"unknown mask format {fmt!r}")
    payload = mask.missing.astype("<u8") if fmt == "indices" else mask.missing_bool.astype(np.uint8)
    payload.tofile(path)
    _put_header(path, {"format": fmt, "dims": [int(d) for d in mask.shape.dims]})


def read_mask(path: str) -> Mask:
    """dataio.py:99-109; the grid is validated first (odd extents raise)."""
    meta = _header(path)
    shape = GridShape(tuple(int(d) for d in meta["dims"]))
    fmt = meta.get("format")
    if fmt not in MASK_FORMATS:
        raise ValueError(f"malformed mask header: unknown format {fmt!r}")
    if fmt == "indices":
        return Mask(np.fromfile(path, dtype="<u8").astype(np.int64), shape)
    flags = np.fromfile(path, dtype=np.uint8)
    if flags.size != shape.n:
        raise ValueError(f"byte mask {path} has {flags.size} entries, grid expects {shape.n}")
    return Mask.from_bool(flags != 0, shape)
