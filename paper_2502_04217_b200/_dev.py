"""Device plumbing: torch CUDA buffers, the current stream, plan cache.

PyTorch is used only to own device memory and to name the stream; every
arithmetic operation on the solver path is a libfftlasso_b200 kernel.
Functions of the public API accept NumPy arrays (the reference's types --
results come back as NumPy) or CUDA tensors (results stay on the device).
"""

from __future__ import annotations

import atexit
import ctypes
import os

import numpy as np

from . import _lib
from .errors import BackendUnavailableError, UnsupportedShapeError

try:
    import torch
except ImportError as exc:  # pragma: no cover - torch is part of the image
    raise BackendUnavailableError("PyTorch is required for device buffers") from exc

F64 = torch.float64


_available = False
# the raw cudaStream_t of the current stream without building a Stream object
# (a few microseconds per call, ~30 calls per IPM solve of a small problem)
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def device() -> "torch.device":
    global _available
    if not _available:
        if not torch.cuda.is_available():
            raise BackendUnavailableError("no CUDA device: the B200 path has no CPU fallback")
        _available = True
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> ctypes.c_void_p:
    if _raw_stream is not None and _available:
        return ctypes.c_void_p(_raw_stream(torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_dev(x, n: int | None = None, what: str = "vector", scratch=None):
    """Flat contiguous float64 CUDA tensor view/copy of ``x``.

    ``scratch`` (a CUDA float64 tensor) may receive the upload of host data
    instead of a fresh allocation (the solver lends its PCG work buffer).
    """
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.device != dev or t.dtype != F64:
            t = t.to(device=dev, dtype=F64)
        t = t.reshape(-1)
        if not t.is_contiguous():
            t = t.contiguous()
    else:
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
        out = scratch[:a.size] if scratch is not None and scratch.numel() >= a.size else None
        if a.nbytes >= _UPLOAD_MIN:
            t = _upload(a, dev, out)
        elif out is not None:
            t = out.copy_(torch.from_numpy(a))
        else:
            t = torch.from_numpy(a).to(dev)
    if n is not None and t.numel() != n:
        raise UnsupportedShapeError(f"{what} has {t.numel()} entries, expected {n}")
    return t


_UPLOAD_MIN = 32 << 20
# host threads filling pinned staging chunks (NumPy releases the GIL in the copy);
# NumPy-in apply_kkt at 512^3 on the 16-core GPU host: 7.3 (8 threads) -> 8.2 (16)
_POOL_WORKERS = max(4, min(16, os.cpu_count() or 4))
_UPLOAD_CHUNK = 64 << 20
# upload_chunks: 32 pinned 32 MiB staging slots in flight (NumPy-in apply_kkt at
# 512^3 on the 16-core GPU host: 8 x 64 MiB 7.76, 16 x 64 MiB 8.09, 32 x 32 MiB
# 8.50, 32 x 16 MiB 7.46 matvec/s; tools/gpu/e2e_slots_probe.py).  Page-locking
# the caller's arrays in place instead (cudaHostRegister) is no faster: ~43
# GB/s serialised in the driver and ~2.5 GB/s when overlapped with the DMA
# (tools/gpu/host_register_probe2.py).
_UPLOAD_SLOTS = 32
_STAGE_CHUNK = 32 << 20
_pool = None
_side_streams: dict = {}


def _upload(a: np.ndarray, dev, out=None):
    """Host->device copy of a large pageable NumPy array.

    A pageable source forces the driver through its own small bounce buffer
    (~10 GB/s).  Instead, worker threads copy 64 MiB chunks into pinned
    buffers (NumPy releases the GIL in the copy) while each finished chunk
    is already DMA-ing up on a side stream; the current stream then waits
    for the side stream.
    """
    global _pool
    from concurrent.futures import ThreadPoolExecutor

    if _pool is None:
        _pool = ThreadPoolExecutor(max_workers=_POOL_WORKERS, thread_name_prefix="fl-upload")
    if out is None:
        out = torch.empty(a.size, dtype=F64, device=dev)
    stage = torch.empty(a.size, dtype=F64, pin_memory=True)
    hs = stage.numpy()
    step = _UPLOAD_CHUNK // 8
    bounds = [(i, min(a.size, i + step)) for i in range(0, a.size, step)]

    def fill(ab):
        np.copyto(hs[ab[0]:ab[1]], a[ab[0]:ab[1]])
        return ab

    side = _side_streams.get(dev.index)
    if side is None:
        side = _side_streams[dev.index] = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        for lo, hi in _pool.map(fill, bounds):
            out[lo:hi].copy_(stage[lo:hi], non_blocking=True)
    torch.cuda.current_stream(dev).wait_stream(side)
    out.record_stream(side)  # (torch's host allocator tracks the pinned stage itself)
    return out


def upload_chunks(groups, stream):
    """Host->device copies in order, one CUDA event per group, on ``stream``.

    ``groups`` is a list of lists of (host CPU tensor, device tensor, lo, hi):
    element range [lo, hi) of the host tensor goes to the same range of the
    device tensor.  Pinned sources DMA directly; pageable ones (NumPy views)
    are copied into pinned 64 MiB slots by worker threads while earlier
    slots are already in flight (a pageable DMA source crawls through the
    driver's bounce buffer).  Returns the per-group events.
    """
    global _pool
    from concurrent.futures import ThreadPoolExecutor

    if _pool is None:
        _pool = ThreadPoolExecutor(max_workers=_POOL_WORKERS, thread_name_prefix="fl-upload")
    step = _STAGE_CHUNK // 8
    pieces = []  # (group index, src, dst, lo, hi), pageable ones split into slots
    for gi, grp in enumerate(groups):
        for src, dst, lo, hi in grp:
            if src.is_pinned():
                pieces.append((gi, src, dst, lo, hi, None))
            else:
                for a in range(lo, hi, step):
                    pieces.append((gi, src, dst, a, min(hi, a + step), True))
    nslot = _UPLOAD_SLOTS
    slots = [torch.empty(step, dtype=F64, pin_memory=True) for _ in range(nslot)]
    slot_free = [None] * nslot  # event: the DMA out of the slot has finished

    def fill(k, src, lo, hi, ev):
        if ev is not None:
            ev.synchronize()
        np.copyto(slots[k].numpy()[:hi - lo], src.numpy()[lo:hi])

    events = []
    futures = {}
    k = 0
    # prefetch: queue the fills of the first nslot pageable pieces
    staged = [i for i, p in enumerate(pieces) if p[5]]
    order = {i: j % nslot for j, i in enumerate(staged)}
    for j, i in enumerate(staged[:nslot]):
        _, src, _, lo, hi, _ = pieces[i]
        futures[i] = _pool.submit(fill, order[i], src, lo, hi, None)
    nxt = nslot
    with torch.cuda.stream(stream):
        for i, (gi, src, dst, lo, hi, paged) in enumerate(pieces):
            if paged:
                k = order[i]
                futures.pop(i).result()
                dst[lo:hi].copy_(slots[k][:hi - lo], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                slot_free[k] = ev
                if nxt < len(staged):  # refill this slot for a later piece
                    ii = staged[nxt]
                    _, s2, _, l2, h2, _ = pieces[ii]
                    futures[ii] = _pool.submit(fill, order[ii], s2, l2, h2, ev)
                    nxt += 1
            else:
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
            if i + 1 == len(pieces) or pieces[i + 1][0] != gi:
                e = torch.cuda.Event()
                e.record(stream)
                events.append(e)
    return events


def empty(n: int):
    return torch.empty(int(n), dtype=F64, device=device())


def pinned(n: int):
    """Page-locked host doubles (targets of asynchronous device->host copies)."""
    return torch.zeros(int(n), dtype=F64, pin_memory=True)


def zeros(n: int):
    return torch.zeros(int(n), dtype=F64, device=device())


_DOWNLOAD_RING_MIN = 4 << 30


def out(t, like_host: bool):
    """Return ``t`` as NumPy when the caller passed host data.

    The device->host copy lands in page-locked memory from torch's caching
    host allocator (full-bandwidth DMA; freed results are recycled by later
    calls), exposed to the caller as a NumPy view.  Results of 4 GiB and
    more go through a ring of pinned 64 MiB chunks into an ordinary NumPy
    array instead (pinning many GB per call costs seconds).
    """
    if not like_host:
        return t
    if t.numel() * t.element_size() >= _DOWNLOAD_RING_MIN and t.dtype == F64 and t.is_contiguous():
        return _download(t).reshape(tuple(t.shape))
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def _download(t):
    """Device->host through 4 pinned 64 MiB slots; worker threads move each
    landed chunk into the result while later chunks are still in flight."""
    global _pool
    from concurrent.futures import ThreadPoolExecutor

    if _pool is None:
        _pool = ThreadPoolExecutor(max_workers=_POOL_WORKERS, thread_name_prefix="fl-upload")
    flat = t.reshape(-1)
    res = np.empty(flat.numel(), dtype=np.float64)
    step = _UPLOAD_CHUNK // 8
    nslot = 4
    ring = [torch.empty(step, dtype=F64, pin_memory=True) for _ in range(nslot)]
    dev = flat.device
    side = _side_streams.get(dev.index)
    if side is None:
        side = _side_streams[dev.index] = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    pending = [None] * nslot

    def drain(ev, k, lo, hi):
        ev.synchronize()
        np.copyto(res[lo:hi], ring[k].numpy()[:hi - lo])

    for i, lo in enumerate(range(0, flat.numel(), step)):
        hi = min(flat.numel(), lo + step)
        k = i % nslot
        if pending[k] is not None:
            pending[k].result()
        with torch.cuda.stream(side):
            ring[k][:hi - lo].copy_(flat[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        pending[k] = _pool.submit(drain, ev, k, lo, hi)
    for f in pending:
        if f is not None:
            f.result()
    flat.record_stream(side)
    return res


class Plan:
    """Owns one fl_plan (per grid shape and device)."""

    def __init__(self, dims, dev_index: int):
        arr = (ctypes.c_int64 * len(dims))(*dims)
        h = ctypes.c_void_p()
        _lib.call("fl_plan_create", len(dims), arr, dev_index, ctypes.byref(h))
        self.handle = h
        self.dims = tuple(dims)
        self.n = int(np.prod(dims))

    def close(self):
        if self.handle:
            _lib.lib().fl_plan_destroy(self.handle)
            self.handle = None


_plans: dict = {}


def plan_for(dims) -> Plan:
    dev = device()
    key = (tuple(int(d) for d in dims), dev.index)
    p = _plans.get(key)
    if p is None:
        p = Plan(key[0], dev.index)
        _plans[key] = p
    return p


@atexit.register
def _release_plans():  # pragma: no cover - process teardown
    for p in _plans.values():
        try:
            p.close()
        except Exception:
            pass
    _plans.clear()
