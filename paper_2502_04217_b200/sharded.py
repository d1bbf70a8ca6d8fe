"""Slab-sharded 3D operators and IPM solve over P ranks.

Layout (d0 = P a, d1 = P b, all dims even):

* **X-slab** of rank r: rows i0 in [r a, (r+1) a), local shape (a, d1, d2) --
  a contiguous chunk of the global row-major vector.  Every IPM / PCG vector
  lives in X-slabs, so all elementwise work is local.
* **Y-slab** of rank r: i1 in [r b, (r+1) b), local layout (b, d2, d0) -- axis 0
  is local *and contiguous*, so the fused synth/mask/analysis pass of the
  single-GPU path runs unchanged on it.  The mask bits and b_hat are stored
  in this layout.

gram (masking.py:107-118; the per-axis maps commute, fourier.py:14-16):

    X: synth axis 2, synth axis 1  ->  all-to-all X->Y  ->
    Y: synth axis 0 . Z . analyze axis 0 (one fused pass)  ->  all-to-all Y->X  ->
    X: analyze axis 1, analyze axis 2

i.e. the single-GPU pass count (5) plus two transposes.  Scalars (dots, norms,
maxima, minima) are combined with one all-reduce per decision point.

``Comm`` hides the exchange: ``DistComm`` runs one shard per process over
``torch.distributed`` (NCCL on B200s; gloo on CPU), ``LocalComm`` holds all
P shards of a grid in one process (single-GPU emulation of the sharded
algorithm -- no kernel ever waits on another rank).  Every operation below
works on *lists of local shards* (length 1 under DistComm, P under
LocalComm).

Two exchange implementations (``ShardedGrid(..., exchange=...)``, default
``"peer"``):

* ``"peer"`` (default; falls back to ``"a2a"`` if peer buffers cannot be
  set up): ONE kernel per direction stores every element, transposed,
  straight into the owning rank's slab through peer pointers (CUDA IPC
  buffers opened on every rank; NVLink / NVSwitch stores), followed by a
  one-element all-reduce as the stream-ordered barrier.  Per element one
  read and one (remote) write instead of three of each, no send buffer.
  Validated bit-for-bit against ``"a2a"`` with LocalComm on one GPU (where
  the "peer" tables are the local shard buffers); the IPC path itself needs
  two or more GPUs;
* ``"a2a"``: pack kernel -> ``all_to_all_single`` (NCCL) -> unpack kernel.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import NumericalBreakdownError, StalledError, UnsupportedShapeError
from .ipm import FIELDS, IpmConfig, IpmState, IterationRecord, SolveReport, _alpha_from_ratio, next_barrier
from .newton_system import fl_state
from .pcg import PcgConfig

SUM, MAX, MIN = "sum", "max", "min"


# ---------------------------------------------------------------------------
# geometry and communication
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SlabGeometry:
    dims: tuple
    P: int

    def __post_init__(self):
        d0, d1, d2 = self.dims
        if any(d < 2 or d % 2 for d in self.dims):
            raise UnsupportedShapeError("every axis must be even and >= 2")
        if d0 % self.P or d1 % self.P:
            raise UnsupportedShapeError(f"slab sharding needs d0 and d1 divisible by P={self.P}")

    @property
    def a(self):
        return self.dims[0] // self.P

    @property
    def b(self):
        return self.dims[1] // self.P

    @property
    def n_local(self):
        return self.dims[0] * self.dims[1] * self.dims[2] // self.P

    @property
    def n(self):
        return self.dims[0] * self.dims[1] * self.dims[2]

    # host-side layout helpers (input scatter / result gather, tests)
    def x_slab(self, full: np.ndarray, r: int) -> np.ndarray:
        return full.reshape(-1)[r * self.n_local:(r + 1) * self.n_local]

    def y_slab(self, full: np.ndarray, r: int) -> np.ndarray:
        d0, d1, d2 = self.dims
        g = full.reshape(d0, d1, d2)[:, r * self.b:(r + 1) * self.b, :]  # (d0, b, d2)
        return np.ascontiguousarray(np.transpose(g, (1, 2, 0))).reshape(-1)  # (b, d2, d0)

    def from_x(self, slabs) -> np.ndarray:
        return np.concatenate([np.asarray(s).reshape(-1) for s in slabs])


class Comm:
    """Exchange interface over the shards held by this process."""

    world: int
    ranks: list  # global rank of each local shard

    def all_to_all(self, send: list) -> list:
        raise NotImplementedError

    def reduce(self, values: list, op: str) -> np.ndarray:
        raise NotImplementedError

    def barrier(self):
        """Stream-ordered cross-rank barrier (after a peer exchange)."""
        raise NotImplementedError

    def reduce_device(self, tensors: list):
        """In-place SUM of small device tensors across ranks, stream ordered,
        no host synchronisation (one tensor per local shard)."""
        raise NotImplementedError

    def peer_buffers(self, n: int):
        """Exchange buffers of ``n`` doubles: (local tensors, pointer tables),
        one per local shard; table[r] addresses rank r's buffer."""
        raise NotImplementedError


class LocalComm(Comm):
    """All P shards in this process: exchanges are block copies."""

    def __init__(self, P: int):
        self.world = P
        self.ranks = list(range(P))

    def all_to_all(self, send):
        P = self.world
        blk = send[0].numel() // P
        recv = [s.new_empty(s.shape) for s in send]
        for dst in range(P):
            for src in range(P):
                recv[dst][src * blk:(src + 1) * blk].copy_(send[src][dst * blk:(dst + 1) * blk])
        return recv

    def reduce(self, values, op):
        arr = np.array([np.asarray(v, dtype=np.float64).reshape(-1) for v in values])
        return {SUM: arr.sum(0), MAX: arr.max(0), MIN: arr.min(0)}[op]

    def barrier(self):
        pass  # one stream: the exchange kernels already ran in order

    def reduce_device(self, tensors):
        # NumPy's summation order over the shards (sequential below 8, the
        # 8-way pairwise tree at 8), on the device
        t = list(tensors)
        if len(t) == 8:
            acc = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]))
        else:
            acc = t[0].clone()
            for x in t[1:]:
                acc = acc + x
        for x in t:
            x.copy_(acc)

    def peer_buffers(self, n):
        bufs = [_dev.empty(n) for _ in range(self.world)]
        table = (ctypes.c_void_p * self.world)(*(b.data_ptr() for b in bufs))
        return bufs, [table] * self.world


def torch_empty_like(t):
    import torch

    return torch.empty_like(t)


class DistComm(Comm):
    """One shard per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]
        self.device = device

    def all_to_all(self, send):
        (s,) = send
        if self.device is None and s.is_cuda:  # host-side group over GPU slabs
            h = s.cpu()
            r = torch_empty_like(h)
            self.dist.all_to_all_single(r, h, group=self.group)
            return [r.to(s.device)]
        recv = s.new_empty(s.shape)
        self.dist.all_to_all_single(recv, s, group=self.group)
        return [recv]

    def reduce(self, values, op):
        import torch

        (v,) = values
        t = torch.as_tensor(np.asarray(v, dtype=np.float64).reshape(-1),
                            device=self.device if self.device is not None else "cpu")
        rop = {SUM: self.dist.ReduceOp.SUM, MAX: self.dist.ReduceOp.MAX, MIN: self.dist.ReduceOp.MIN}[op]
        self.dist.all_reduce(t, op=rop, group=self.group)
        return t.cpu().numpy()

    def barrier(self):
        import torch

        # an all-reduce cannot complete on any rank before every rank's stream
        # reached it, i.e. before every rank's exchange kernel has finished
        # (NCCL: stream-ordered).  A host-side group (gloo) over GPU data orders
        # nothing on the device, so the stream is drained first.
        if self.device is None and torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.current_stream().synchronize()
        t = torch.zeros(1, dtype=torch.float64, device=self.device if self.device is not None else "cpu")
        self.dist.all_reduce(t, group=self.group)

    def reduce_device(self, tensors):
        (t,) = tensors
        if self.device is None and t.is_cuda:  # host-side group: reduce a host copy
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
            return
        self.dist.all_reduce(t, group=self.group)

    def peer_buffers(self, n):
        """Collective and all-or-nothing: every rank allocates, the handles are
        all-gathered, every rank opens every peer's buffer; if any rank fails
        at any step, all ranks raise (so they fall back together)."""
        import torch

        dev = self.device if self.device is not None else "cpu"
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        ok = 1
        try:
            _lib.call("fl_ipc_alloc", n * 8, ctypes.byref(ptr), handle)
        except (RuntimeError, MemoryError, OSError):
            ok = 0
        mine = torch.frombuffer(bytearray(handle.raw + bytes([ok])), dtype=torch.uint8).to(dev)
        gathered = [torch.empty(65, dtype=torch.uint8, device=dev) for _ in range(self.world)]
        self.dist.all_gather(gathered, mine, group=self.group)
        got = [g.cpu().numpy().tobytes() for g in gathered]
        me = self.ranks[0]
        ptrs, opened = [], []
        if all(g[64] == 1 for g in got):
            for r, g in enumerate(got):
                if r == me:
                    ptrs.append(ptr.value)
                    continue
                q = ctypes.c_void_p()
                try:
                    _lib.call("fl_ipc_open", g[:64], ctypes.byref(q))
                except (RuntimeError, OSError):
                    ok = 0
                    break
                ptrs.append(q.value)
                opened.append(q.value)
        else:
            ok = 0
        flag = torch.tensor([float(ok)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.group)
        if flag.item() < 1.0:
            for q in opened:
                _lib.call("fl_ipc_close", ctypes.c_void_p(q))
            if ptr.value:
                _lib.call("fl_dev_free", ptr)
            raise RuntimeError("peer buffers unavailable on at least one rank")
        self._opened = getattr(self, "_opened", []) + opened
        self._owned = getattr(self, "_owned", []) + [ptr.value]
        table = (ctypes.c_void_p * self.world)(*ptrs)
        return [_wrap_device(ptr.value, n)], [table]

    def release_peer_buffers(self):
        """Close the peers' IPC mappings and free this rank's exchange buffers
        (collective: every rank calls it once it is done with the grid)."""
        self.dist.barrier(group=self.group)
        for ptr in getattr(self, "_opened", []):
            _lib.call("fl_ipc_close", ctypes.c_void_p(ptr))
        self.dist.barrier(group=self.group)
        for ptr in getattr(self, "_owned", []):
            _lib.call("fl_dev_free", ctypes.c_void_p(ptr))
        self._opened, self._owned = [], []


class _CudaArray:
    """__cuda_array_interface__ view of a raw device allocation (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                          "version": 3, "strides": None}


def _wrap_device(ptr: int, n: int):
    import torch

    return torch.as_tensor(_CudaArray(ptr, n), device=_dev.device())


# ---------------------------------------------------------------------------
# local device operations of one shard (C ABI)
# ---------------------------------------------------------------------------

class ShardOps:
    """Per-shard GPU kernels: X-slab passes, Y-slab fused pass, slab transposes."""

    def __init__(self, geo: SlabGeometry):
        self.geo = geo
        d0, d1, d2 = geo.dims
        dev = _dev.device().index
        self.x_plan = self._plan((geo.a, d1, d2), 0b110, dev)
        self.y_plan = self._plan((geo.b, d2, d0), 0b100, dev)

    @staticmethod
    def _plan(dims, mask, dev):
        arr = (ctypes.c_int64 * 3)(*dims)
        h = ctypes.c_void_p()
        _lib.call("fl_plan_create_ex", 3, arr, mask, dev, ctypes.byref(h))
        return h

    # buffers of this backend
    @staticmethod
    def empty(n):
        return _dev.empty(n)

    @staticmethod
    def vec(a):
        return _dev.to_dev(a)

    @staticmethod
    def bits(flags):
        import torch

        return torch.from_numpy(pack_bits(flags)).to(_dev.device())

    def close(self):
        for h in (self.x_plan, self.y_plan, *self.__dict__.get("_chunk_plans", {}).values()):
            if h:
                _lib.lib().fl_plan_destroy(h)
        self.x_plan = self.y_plan = None
        self.__dict__.pop("_chunk_plans", None)

    def synth_x(self, src, dst):  # axes 2 then 1 of the X-slab
        _lib.call("fl_axis_pass", self.x_plan, 2, 0, _dev.ptr(src), _dev.ptr(dst), _dev.stream())
        _lib.call("fl_axis_pass", self.x_plan, 1, 0, _dev.ptr(dst), _dev.ptr(dst), _dev.stream())

    def analyze_x(self, src, dst):
        _lib.call("fl_axis_pass", self.x_plan, 1, 1, _dev.ptr(src), _dev.ptr(dst), _dev.stream())
        _lib.call("fl_axis_pass", self.x_plan, 2, 1, _dev.ptr(dst), _dev.ptr(dst), _dev.stream())

    def synth_y0(self, src, dst):  # axis 0 of the grid = contiguous axis of the Y-slab
        _lib.call("fl_axis_pass", self.y_plan, 2, 0, _dev.ptr(src), _dev.ptr(dst), _dev.stream())

    def fused_y(self, bits, bhat, src, dst, want_norm: bool):
        nrm = ctypes.c_double(0.0)
        _lib.call("fl_fused_mask_pass", self.y_plan, _dev.ptr(bits), _dev.ptr(bhat) if bhat is not None else None,
                  _dev.ptr(src), _dev.ptr(dst), ctypes.byref(nrm) if want_norm else None, _dev.stream())
        return nrm.value

    def fused_y_dev(self, bits, src, dst, nrm_dev):
        """Fused gram pass with ||Z A beta||^2 (local) written to device memory."""
        _lib.call("fl_fused_mask_pass_dev", self.y_plan, _dev.ptr(bits), _dev.ptr(src), _dev.ptr(dst),
                  ctypes.c_void_p(nrm_dev.data_ptr()), _dev.stream())

    def pack_x(self, x, send):
        g = self.geo
        _lib.call("fl_slab_pack_x", g.a, g.dims[1], g.dims[2], g.P, _dev.ptr(x), _dev.ptr(send), _dev.stream())

    def unpack_y(self, recv, y):
        g = self.geo
        _lib.call("fl_slab_unpack_y", g.a, g.b, g.dims[2], g.P, _dev.ptr(recv), _dev.ptr(y), _dev.stream())

    def pack_y(self, y, send):
        g = self.geo
        _lib.call("fl_slab_pack_y", g.a, g.b, g.dims[2], g.P, _dev.ptr(y), _dev.ptr(send), _dev.stream())

    def unpack_x(self, recv, x):
        g = self.geo
        _lib.call("fl_slab_unpack_x", g.a, g.dims[1], g.dims[2], g.P, _dev.ptr(recv), _dev.ptr(x), _dev.stream())

    def synth_x_planes(self, src, dst, i0, count):
        """synth_x on planes [i0, i0 + count) only (for the overlapped exchange)."""
        g = self.geo
        key = int(count)
        plans = self.__dict__.setdefault("_chunk_plans", {})
        if key not in plans:
            plans[key] = self._plan((key, g.dims[1], g.dims[2]), 0b110, _dev.device().index)
        off = int(i0) * g.dims[1] * g.dims[2] * 8
        s_ = ctypes.c_void_p(src.data_ptr() + off)
        d_ = ctypes.c_void_p(dst.data_ptr() + off)
        _lib.call("fl_axis_pass", plans[key], 2, 0, s_, d_, _dev.stream())
        _lib.call("fl_axis_pass", plans[key], 1, 0, d_, d_, _dev.stream())

    def x_to_y_peers_planes(self, rank, x, table, i0, count):
        g = self.geo
        off = int(i0) * g.dims[1] * g.dims[2] * 8
        _lib.call("fl_slab_x_to_y_peers_planes", g.a, g.dims[1], g.dims[2], g.P, rank, int(i0), int(count),
                  ctypes.c_void_p(x.data_ptr() + off), ctypes.cast(table, ctypes.POINTER(ctypes.c_void_p)),
                  _dev.stream())

    def x_to_y_peers(self, rank, x, table):
        g = self.geo
        _lib.call("fl_slab_x_to_y_peers", g.a, g.dims[1], g.dims[2], g.P, rank, _dev.ptr(x),
                  ctypes.cast(table, ctypes.POINTER(ctypes.c_void_p)), _dev.stream())

    def y_to_x_peers(self, rank, y, table):
        g = self.geo
        _lib.call("fl_slab_y_to_x_peers", g.a, g.b, g.dims[2], g.P, rank, _dev.ptr(y),
                  ctypes.cast(table, ctypes.POINTER(ctypes.c_void_p)), _dev.stream())


# ---------------------------------------------------------------------------
# sharded operators
# ---------------------------------------------------------------------------

class ShardedGrid:
    """Geometry, comm, per-shard ops and exchange buffers of one sharded grid."""

    def __init__(self, dims, comm: Comm, ops_factory=ShardOps, exchange=None, chunks=None):
        self.geo = SlabGeometry(tuple(int(d) for d in dims), comm.world)
        self.comm = comm
        self.ops = [ops_factory(self.geo) for _ in comm.ranks]
        n = self.geo.n_local
        # forward exchange in plane chunks overlapped with the X-side passes:
        # default 4 with two or more real ranks, off on one GPU
        self.chunks = chunks
        self.exchange = exchange or "peer"
        if self.exchange not in ("a2a", "peer"):
            raise ValueError(f"unknown exchange {self.exchange!r}")
        if self.exchange == "peer":
            # grid-owned receive slabs, addressable by every rank
            try:
                self.ybuf, self.ytab = comm.peer_buffers(n)
                self.xrecv, self.xtab = comm.peer_buffers(n)
            except (RuntimeError, OSError, ValueError, AttributeError, MemoryError) as exc:
                if exchange == "peer":  # explicitly requested: do not hide the failure
                    raise
                import warnings

                warnings.warn(f"peer exchange unavailable ({exc}); using all-to-all")
                self.exchange = "a2a"
        if self.exchange == "a2a":
            self.send = [self.ops[0].empty(n) for _ in comm.ranks]
            self.ybuf = [self.ops[0].empty(n) for _ in comm.ranks]

    def x_to_y(self, xs, ys):
        if self.exchange == "peer":  # into the grid's Y slabs, then copy if asked elsewhere
            for i, (op, r, x) in enumerate(zip(self.ops, self.comm.ranks, xs)):
                op.x_to_y_peers(r, x, self.ytab[i])
            self.comm.barrier()
            for y, yb in zip(ys, self.ybuf):
                if y.data_ptr() != yb.data_ptr():
                    y.copy_(yb)
            return
        for op, x, s in zip(self.ops, xs, self.send):
            op.pack_x(x, s)
        recv = self.comm.all_to_all(self.send)
        for op, rv, y in zip(self.ops, recv, ys):
            op.unpack_y(rv, y)

    def y_to_x(self, ys, xs):
        """Y slabs -> X slabs; with the peer exchange the result lands in the
        grid's receive slabs (returned), otherwise in ``xs``."""
        if self.exchange == "peer":
            for i, (op, r, y) in enumerate(zip(self.ops, self.comm.ranks, ys)):
                op.y_to_x_peers(r, y, self.xtab[i])
            self.comm.barrier()
            return self.xrecv
        for op, y, s in zip(self.ops, ys, self.send):
            op.pack_y(y, s)
        recv = self.comm.all_to_all(self.send)
        for op, rv, x in zip(self.ops, recv, xs):
            op.unpack_x(rv, x)
        return xs

    def _overlapped_forward(self, betas, outs) -> bool:
        """synth_x + X->Y exchange in plane chunks, the exchange of chunk c on a
        side stream while chunk c+1 is transformed (peer exchange only).

        Default: 4 chunks with two or more ranks (the NVLink stores overlap the
        next chunk's passes); off for one rank / LocalComm, where both compete
        for the same SMs and HBM (measured: 194 -> 187 matvecs/s at 512^3, P = 1).
        ``ShardedGrid(chunks=K)`` overrides; the chunked path is tested in emulation.
        """
        K = self.chunks if self.chunks is not None else (
            4 if isinstance(self.comm, DistComm) and self.comm.world > 1 else 1)
        a = self.geo.a
        if self.exchange != "peer" or K <= 1 or a % K or not hasattr(self.ops[0], "synth_x_planes"):
            return False
        import torch

        main = torch.cuda.current_stream()
        side = self.__dict__.get("_xstream")
        if side is None:
            side = self._xstream = torch.cuda.Stream(main.device)
        side.wait_stream(main)
        ac = a // K
        for i, (op, r, b, o) in enumerate(zip(self.ops, self.comm.ranks, betas, outs)):
            for c in range(K):
                op.synth_x_planes(b, o, c * ac, ac)
                ev = torch.cuda.Event()
                ev.record(main)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    op.x_to_y_peers_planes(r, o, self.ytab[i], c * ac, ac)
        main.wait_stream(side)
        for o in outs:
            o.record_stream(side)
        self.comm.barrier()
        return True

    def synthesize_to_y(self, betas, ys):
        """A beta with beta in X-slabs; result in Y-slabs (b, d2, d0)."""
        scratch = self.xrecv if self.exchange == "peer" else self.ybuf
        for op, b, x in zip(self.ops, betas, scratch):
            op.synth_x(b, x)  # X-layout scratch
        self.x_to_y(scratch, ys)
        for op, y in zip(self.ops, ys):
            op.synth_y0(y, y)

    def gram(self, betas, outs, bits_y, bhat_y=None, want_norm=False, extra=None, norm_dev=None):
        """outs = A^T Z A beta (bhat_y None) or A^T Z (b_hat - A beta); X-slabs in/out.

        Returns the all-reduced ||Z A beta||^2 when ``want_norm`` (gram only);
        with ``extra`` (one local partial per shard) the same all-reduce also
        sums those and returns (norm, extra_sum).  With ``norm_dev`` (one
        device scalar per shard) the LOCAL norm goes there instead, with no
        host synchronisation (the device-scalar PCG reduces it itself).
        """
        if not self._overlapped_forward(betas, outs):
            for op, b, o in zip(self.ops, betas, outs):
                op.synth_x(b, o)
            self.x_to_y(outs, self.ybuf)
        norms = []
        for i, (op, y) in enumerate(zip(self.ops, self.ybuf)):
            if norm_dev is not None:
                op.fused_y_dev(bits_y[i], y, y, norm_dev[i])
                continue
            norms.append(op.fused_y(bits_y[i], None if bhat_y is None else bhat_y[i], y, y, want_norm))
        src = self.y_to_x(self.ybuf, outs)
        for op, x, o in zip(self.ops, src, outs):
            op.analyze_x(x, o)
        if want_norm:
            if extra is not None:
                red = self.comm.reduce([[v, e] for v, e in zip(norms, extra)], SUM)
                return float(red[0]), float(red[1])
            return float(self.comm.reduce([[v] for v in norms], SUM)[0])
        return None


def kkt_apply(grid: ShardedGrid, bits_y, sig1, sig2, d_betas, d_zs, tops, bots, want_pkp=False):
    """Sharded condensed KKT matvec (newton_system.py:148-152) on X-slabs.

    Sharded gram, then the local elementwise epilogue on every slab; returns
    the all-reduced d.Kd when ``want_pkp``.
    """
    grid.gram(d_betas, tops, bits_y)
    L = _lib.lib()
    parts = []
    for i, (t, b, db, dz) in enumerate(zip(tops, bots, d_betas, d_zs)):
        v = ctypes.c_double()
        _lib.check(L.fl_kkt_epilogue(grid.geo.n_local, _dev.ptr(t), _dev.ptr(db), _dev.ptr(dz), _dev.ptr(sig1[i]),
                                     _dev.ptr(sig2[i]), _dev.ptr(b), ctypes.byref(v) if want_pkp else None,
                                     _dev.stream()))
        parts.append([v.value])
    return float(grid.comm.reduce(parts, SUM)[0]) if want_pkp else None


def bragg_y_flags(geo: SlabGeometry, r: int, spacing: int = 16, radius: float = 5.3) -> np.ndarray:
    """Bragg punch mask (workloads.bragg_flags) generated directly in rank r's
    Y-slab layout (b, d2, d0) -- no full-grid host array for C5-sized grids."""
    d0, d1, d2 = geo.dims
    def sq(m):
        t = np.arange(m) % spacing
        return np.minimum(t, spacing - t).astype(np.int64) ** 2
    s0, s1, s2 = sq(d0), sq(d1)[r * geo.b:(r + 1) * geo.b], sq(d2)
    tot = s1[:, None, None] + s2[None, :, None] + s0[None, None, :]
    return (tot <= radius * radius).reshape(-1)


# ---------------------------------------------------------------------------
# sharded IPM solve (ipm.py:402-486 over slabs)
# ---------------------------------------------------------------------------

def _st(st):
    return ctypes.byref(fl_state(st))


class ShardedProblem:
    """Per-shard device data of one instance: Y-layout mask bits and b_hat."""

    def __init__(self, grid: ShardedGrid, bits_y, bhat_y):
        self.grid = grid
        self.bits_y = bits_y
        self.bhat_y = bhat_y

    @classmethod
    def from_host(cls, grid: ShardedGrid, flags: np.ndarray, b_hat_full: np.ndarray):
        """Scatter a host problem (full-grid missing flags, embedded b) to this process's shards."""
        bits, bh = [], []
        for r in grid.comm.ranks:
            bits.append(grid.ops[0].bits(grid.geo.y_slab(np.asarray(flags, dtype=np.uint8), r)))
            bh.append(grid.ops[0].vec(grid.geo.y_slab(np.asarray(b_hat_full, dtype=np.float64), r)))
        return cls(grid, bits, bh)


def c4_problem_device(grid: ShardedGrid, noise_seed: int = 0, spacing: int = 16, radius: float = 5.3):
    """The C4/C5 recipe built on the devices straight into slab layout
    (no full-grid host array) -> (ShardedProblem, idx, val, lam).

    Same input as ``workloads.c4_const_device`` on one GPU: the recipe's
    spikes (``workloads.c4_spikes``) scattered into each X-slab, the sharded
    synthesis to Y-slabs, then ``fl_noisy_embed`` in Y layout -- the noise is
    a function of the global voxel index, so b_hat is the single-GPU one up
    to the transforms' rounding (their axis order differs).  The Y-slab mask
    is the Bragg mask of the local box (b, d2, d0) when b is a multiple of
    ``spacing`` (the periodic distance of i1 = r b + j1 is then that of j1),
    else the host formula (``bragg_y_flags``).
    """
    import torch

    from . import workloads

    geo = grid.geo
    d0, d1, d2 = geo.dims
    nl = geo.n_local
    idx, val = workloads.c4_spikes(geo.n)
    idx_t = torch.from_numpy(idx).to(_dev.device())
    val_t = torch.from_numpy(val).to(_dev.device())
    betas, bits = [], []
    for r in grid.comm.ranks:
        bx = _dev.empty(nl)
        bx.zero_()
        sel = (idx_t >= r * nl) & (idx_t < (r + 1) * nl)
        bx[idx_t[sel] - r * nl] = val_t[sel]
        betas.append(bx)
        if geo.b % spacing == 0:
            nw = (nl + 31) // 32
            w = torch.empty(nw, dtype=torch.int32, device=_dev.device())
            offs = torch.empty(nw, dtype=torch.int64, device=_dev.device())
            dims = (ctypes.c_int64 * 3)(geo.b, d2, d0)
            n_obs = ctypes.c_int64()
            _lib.call("fl_mask_bragg", 3, dims, int(spacing), float(radius), _dev.ptr(w), _dev.ptr(offs),
                      ctypes.byref(n_obs), _dev.stream())
            del offs
            bits.append(w)
        else:
            bits.append(grid.ops[0].bits(bragg_y_flags(geo, r, spacing, radius)))
    ys = [_dev.empty(nl) for _ in grid.comm.ranks]
    grid.synthesize_to_y(betas, ys)
    del betas
    for i, r in enumerate(grid.comm.ranks):
        # Y-slab local box (b, d2, d0) = global (i1 = r b + j1, i2, i0)
        workloads.noisy_embed_device(ys[i], bits[i], (geo.b, d2, d0), (r * geo.b, 0, 0), (d2, 1, d1 * d2),
                                     noise_seed)
    return ShardedProblem(grid, bits, ys), idx, val, 0.5


def gather_support(betas, geo: SlabGeometry, comm: Comm, rel: float = 1e-6):
    """Global indices of |beta| > rel * max|beta| over all slabs (diagnostics
    classify_support threshold) -> sorted int64 array on every process."""
    import torch

    mx = float(comm.reduce([[float(b.abs().max())] for b in betas], MAX)[0])
    thr = rel * mx
    local = [torch.nonzero(b.abs() > thr).flatten().cpu().numpy() + r * geo.n_local
             for b, r in zip(betas, comm.ranks)]
    if isinstance(comm, DistComm):
        import torch.distributed as dist

        out = [None] * comm.world
        dist.all_gather_object(out, local[0], group=comm.group)
        local = out
    return np.sort(np.concatenate(local)) if local else np.zeros(0, np.int64)


def pack_bits(flags: np.ndarray) -> np.ndarray:
    """Missing flags -> little-endian 32-bit words (bit v & 31 of word v >> 5)."""
    pad = (-flags.size) % 32
    fb = np.concatenate([np.asarray(flags, dtype=np.uint8).reshape(-1), np.zeros(pad, np.uint8)])
    return np.packbits(fb, bitorder="little").view(np.int32).copy()


def sharded_solve(prob: ShardedProblem, lam: float, config: IpmConfig = IpmConfig(), observer=None):
    """Interior-point solve over slabs; returns (beta X-slabs, SolveReport).

    Same control flow, scalars and records as ipm.solve; every scalar decision
    uses one all-reduce of the local kernel reductions.
    """
    grid = prob.grid
    comm = grid.comm
    nl = grid.geo.n_local
    n = grid.geo.n
    S = len(comm.ranks)
    L = _lib.lib()
    s = _dev.stream()
    ws = [_Work(nl) for _ in range(S)]
    mu = lam / 2.0 if config.mu_init is None else float(config.mu_init)
    for w in ws:
        _lib.check(L.fl_ipm_init(nl, _st(w.state), float(lam), s))

    def resid():
        grid.gram([w.state.beta for w in ws], [w.g for w in ws], prob.bits_y, prob.bhat_y)

    def assess(mu_):
        vals = []
        for w in ws:
            a = _lib.FlAssess()
            _lib.check(L.fl_ipm_assess(nl, _st(w.state), _dev.ptr(w.g), float(lam), float(mu_), ctypes.byref(a), s))
            vals.append([a.stationarity, a.dual_equality, a.multiplier_gap, a.primal, a.complementarity,
                         a.barrier_residual, a.min_product, a.dot_nu_s1, a.dot_nu_s2])
        mx = comm.reduce([v[:6] for v in vals], MAX)
        mn = comm.reduce([v[6:7] for v in vals], MIN)
        sm = comm.reduce([v[7:9] for v in vals], SUM)
        worst = max(mx[:5])
        measure = float(sm[0] + sm[1]) / (2 * n)
        return dict(stationarity=mx[0], dual_equality=mx[1], multiplier_gap=mx[2], primal=mx[3],
                    complementarity=mx[4], max_residual=worst, converged=worst <= config.tol,
                    centrality_ok=bool(mn[0] >= config.gamma_centrality * measure),
                    barrier_residual=mx[5], duality_measure=measure)

    t0 = time.perf_counter()
    records = []
    best_kkt = math.inf
    for w in ws:
        w.best.copy_(w.state.beta)
    status = "max_iters"
    resid()
    conv = assess(mu)
    for iteration in range(1, config.max_iters + 1):
        if conv["converged"]:
            status = "converged"
            break
        if conv["barrier_residual"] <= config.inner_slack * mu:
            mu = next_barrier(mu, config.tol, config)
        t_iter = time.perf_counter()
        bad = []
        for w in ws:
            st = L.fl_barrier_diagonals(nl, *(_dev.ptr(getattr(w.state, f)) for f in ("s1", "s2", "nu1", "nu2")),
                                        _dev.ptr(w.sig1), _dev.ptr(w.sig2), None, None, None, None, s)
            bad.append([0.0 if st == 0 else 1.0])
            if st not in (0, _lib.FL_E_INTERIOR):
                _lib.check(st)
            _lib.check(L.fl_newton_rhs(nl, _st(w.state), _dev.ptr(w.g), _dev.ptr(w.sig1), _dev.ptr(w.sig2),
                                       float(lam), float(mu), None, None, None, None, None, None,
                                       _dev.ptr(w.rhs[:nl]), _dev.ptr(w.rhs[nl:]), s))
        if comm.reduce(bad, MAX)[0]:
            from .errors import InteriorViolationError
            raise InteriorViolationError("slacks and multipliers must be strictly positive and finite")
        iters, res_norm = _sharded_pcg(grid, prob, ws, PcgConfig(abs_tol=config.cg_tol, max_iters=config.cg_max_iters))
        tau = max(config.ftb_tau, 1.0 - mu)
        ratios = []
        for w in ws:
            rr = (ctypes.c_double * 4)()
            _lib.check(L.fl_ipm_ratios(nl, _st(w.state), _dev.ptr(w.sig1), _dev.ptr(w.sig2), float(mu),
                                       _dev.ptr(w.x[:nl]), _dev.ptr(w.x[nl:]), rr, s))
            ratios.append(list(rr))
        rmin = comm.reduce(ratios, MIN)
        alpha_p = min(_alpha_from_ratio(rmin[0], tau), _alpha_from_ratio(rmin[1], tau))
        alpha_d = min(_alpha_from_ratio(rmin[2], tau), _alpha_from_ratio(rmin[3], tau))
        if min(alpha_p, alpha_d) < 1e-12:
            raise StalledError(f"fraction-to-boundary step collapsed (alpha_p={alpha_p:.2e}, alpha_d={alpha_d:.2e})")
        stalled = []
        for w in ws:
            st = L.fl_ipm_update(nl, _st(w.state), _dev.ptr(w.sig1), _dev.ptr(w.sig2), float(mu),
                                 _dev.ptr(w.x[:nl]), _dev.ptr(w.x[nl:]), float(alpha_p), float(alpha_d), s)
            if st not in (0, _lib.FL_E_STALLED):
                _lib.check(st)
            stalled.append([1.0 if st == _lib.FL_E_STALLED else 0.0])
        if comm.reduce(stalled, MAX)[0]:
            raise StalledError("slack or multiplier left the strict interior")
        resid()
        conv = assess(mu)
        rec = IterationRecord(iteration=iteration, mu=mu, primal_inf=conv["primal"],
                              dual_inf=max(conv["dual_equality"], conv["multiplier_gap"], conv["stationarity"]),
                              complementarity=conv["complementarity"], kkt_max=conv["max_residual"],
                              krylov_iters=iters, alpha_primal=alpha_p, alpha_dual=alpha_d,
                              pcg_residual=res_norm, centrality_ok=conv["centrality_ok"],
                              wall_time=time.perf_counter() - t_iter)
        records.append(rec)
        if conv["max_residual"] < best_kkt:
            best_kkt = conv["max_residual"]
            for w in ws:
                w.best.copy_(w.state.beta)
        if observer is not None:
            observer([w.state for w in ws], rec)
    else:
        if conv["converged"]:
            status = "converged"
    betas = [w.state.beta if status == "converged" else w.best for w in ws]
    # objective: x = A beta in Y-slabs against b_hat / mask in the same layout
    terms = []
    for w in ws:
        w.g.zero_()
    grid.synthesize_to_y(betas, [w.g for w in ws])
    for i, w in enumerate(ws):
        out = (ctypes.c_double * 2)()
        _lib.check(L.fl_objective_terms(nl, _dev.ptr(prob.bits_y[i]), _dev.ptr(prob.bhat_y[i]), _dev.ptr(w.g), nl,
                                        _dev.ptr(betas[i]), out, s))
        terms.append([out[0], out[1]])
    t = comm.reduce(terms, SUM)
    report = SolveReport(status=status, iterations=len(records), lam=lam, tol=config.tol, records=records,
                         final_objective=0.5 * float(t[0]) + lam * float(t[1]),
                         final_kkt=conv["max_residual"] if status == "converged" else best_kkt,
                         final_mu=mu, wall_time=time.perf_counter() - t0)
    return betas, report


class _Work:
    def __init__(self, nl):
        self.state = IpmState(mu=0.0, **{f: _dev.empty(nl) for f in FIELDS})
        self.sig1, self.sig2, self.g, self.best = (_dev.empty(nl) for _ in range(4))
        self.rhs, self.x, self.r, self.p = (_dev.empty(2 * nl) for _ in range(4))
        self.gp = _dev.empty(nl)


def _sharded_pcg(grid: ShardedGrid, prob: ShardedProblem, ws, cfg: PcgConfig):
    """PCG v2 over slabs (pcg.py:57-127): curvature = ||Z A p_beta||^2 + diagonal form.

    Device scalars: the fused pass leaves the local ||Z A p||^2 on the
    device, the two all-reduces of an iteration (curvature, r'P^{-1}r) run on
    device buffers in stream order (``Comm.reduce_device``: NCCL between
    GPUs), alpha = rho / curv is formed on the device (``fl_pcg_step_alpha``,
    the host's operation order) and read by the update kernel; the host
    synchronises ONCE per iteration, to read (curv, rho') for pcg.py's
    breakdown checks and stopping test (it was five synchronisations: three
    kernel partials and two all-reduces).
    """
    import torch

    comm = grid.comm
    nl = grid.geo.n_local
    L = _lib.lib()
    s = _dev.stream()
    limit = cfg.iteration_limit(2 * grid.geo.n)
    parts = []
    for w in ws:
        out = (ctypes.c_double * 2)()
        _lib.check(L.fl_pcg_step_init(nl, _dev.ptr(w.sig1), _dev.ptr(w.sig2), _dev.ptr(w.rhs), _dev.ptr(w.x),
                                      _dev.ptr(w.r), _dev.ptr(w.p), out, s))
        parts.append([out[0], out[1]])
    rho = float(comm.reduce([[p_[0]] for p_ in parts], SUM)[0])
    if not math.isfinite(rho) or rho < 0:
        raise NumericalBreakdownError(f"preconditioner produced r'P^{{-1}}r = {rho}")
    norm = math.sqrt(rho)
    thr = cfg.abs_tol + cfg.rel_tol * norm
    if norm <= thr:
        return 0, norm
    # per shard: [0] ||Z A p||^2 (local -> global), [1] p.(K-G)p (local -> global),
    # [2] curv, [3] alpha, [4] rho, [5] rho' (local -> global)
    slots = [torch.zeros(8, dtype=torch.float64, device=_dev.device()) for _ in ws]
    for sl, p_ in zip(slots, parts):
        sl[1] = p_[1]
        sl[4] = rho
    for k in range(1, limit + 1):
        grid.gram([w.p[:nl] for w in ws], [w.gp for w in ws], prob.bits_y, norm_dev=[sl[0:1] for sl in slots])
        comm.reduce_device([sl[0:2] for sl in slots])
        for w, sl in zip(ws, slots):
            _lib.check(L.fl_pcg_step_alpha(ctypes.c_void_p(sl.data_ptr()), ctypes.c_void_p(sl.data_ptr() + 32),
                                           ctypes.c_void_p(sl.data_ptr() + 16), s))
            _lib.check(L.fl_pcg_step_update_dev(nl, _dev.ptr(w.sig1), _dev.ptr(w.sig2),
                                                ctypes.c_void_p(sl.data_ptr() + 24), _dev.ptr(w.x), _dev.ptr(w.r),
                                                _dev.ptr(w.p), _dev.ptr(w.gp), ctypes.c_void_p(sl.data_ptr() + 40),
                                                s))
        comm.reduce_device([sl[5:6] for sl in slots])
        h = slots[0][2:6].cpu().numpy()  # the iteration's one synchronisation
        curv, rho_next = float(h[0]), float(h[3])
        if not math.isfinite(curv) or curv <= 0:
            raise NumericalBreakdownError(f"nonpositive curvature p'Kp = {curv} at iteration {k}")
        if not math.isfinite(rho_next) or rho_next < 0:
            raise NumericalBreakdownError(f"r'P^{{-1}}r = {rho_next} at iteration {k}")
        norm = math.sqrt(rho_next)
        if norm <= thr:
            return k, norm
        beta = rho_next / rho
        for w, sl in zip(ws, slots):
            _lib.check(L.fl_pcg_step_pupdate_dev(nl, _dev.ptr(w.sig1), _dev.ptr(w.sig2), _dev.ptr(w.r), float(beta),
                                                 _dev.ptr(w.p), ctypes.c_void_p(sl.data_ptr() + 8), s))
            sl[4:5].copy_(sl[5:6])
        rho = rho_next
    raise NumericalBreakdownError(f"PCG stalled at preconditioned residual {norm:.3e} after {limit} iterations")


# ---------------------------------------------------------------------------
# drop-in entry: solve(b, mask, config, observer) over slab-sharded ranks
# ---------------------------------------------------------------------------

def default_comm() -> Comm:
    """DistComm over the default process group when torch.distributed is
    initialised (one rank per GPU), else a single local shard."""
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return DistComm(device=_dev.device() if dist.get_backend() == "nccl" else None)
    except Exception:  # pragma: no cover - torch.distributed unavailable
        pass
    return LocalComm(1)


def _y_inputs(geo: SlabGeometry, flags: np.ndarray, b_hat: np.ndarray, r: int):
    """Rank r's Y-slab mask bits and b_hat (host transposes of the full grid)."""
    return pack_bits(geo.y_slab(flags.astype(np.uint8), r)), geo.y_slab(b_hat, r)


def solve(b, mask, config: IpmConfig = IpmConfig(), observer=None, comm: Comm | None = None, root: int = 0):
    """``ipm.solve`` (reference ipm.py:402-486) over P slab-sharded GPUs.

    The reference's calling convention on the ``root`` rank: ``b`` the
    observed samples (NumPy, n_observed) and ``mask`` a 3D ``Mask`` (or
    ``BraggMask``); the other ranks pass ``None`` for both.  Root embeds b on
    the full grid, cuts every rank's Y-slab (axis 0 local and contiguous) of
    b_hat and of the mask, and ships them over the process group (NCCL
    point-to-point on B200s); every rank then runs ``sharded_solve`` on its
    slabs (5 HBM passes + 2 slab exchanges per gram, one all-reduce per
    scalar decision).  The default penalty 0.1 max|M^T b| (ipm.py:204-206)
    comes from one sharded residual pass at beta = 0.

    Returns ``(beta, report)`` on root -- beta gathered into one NumPy vector
    (X-slabs are contiguous chunks of the global vector) -- and
    ``(None, report)`` elsewhere; the report is identical on every rank.
    """
    import torch

    comm = comm or default_comm()
    dist_mode = isinstance(comm, DistComm)
    me = comm.ranks[0]
    is_root = (not dist_mode) or me == root
    if is_root:
        if mask.shape.ndim != 3:
            raise UnsupportedShapeError("the sharded solver takes 3D grids")
        meta = [tuple(mask.shape.dims), config]
    else:
        meta = [None, None]
    if dist_mode:
        comm.dist.broadcast_object_list(meta, src=root, group=comm.group)
    dims, config = meta
    if config.lam is not None and config.lam <= 0:
        raise ValueError("penalty must be positive")
    grid = ShardedGrid(dims, comm)
    geo = grid.geo
    nl = geo.n_local
    dev = _dev.device()
    bits, bhat = {}, {}
    # tensors on the wire live where the group's backend wants them: the GPU
    # for NCCL, host memory for a host-side group (gloo)
    wire = dev if (not dist_mode or getattr(comm, "device", None) is not None) else torch.device("cpu")
    if is_root:
        flags = np.asarray(mask.missing_bool, dtype=bool).reshape(-1)
        bv = b.detach().cpu().numpy() if _dev.is_device(b) else np.asarray(b, dtype=np.float64).reshape(-1)
        if bv.size != int((~flags).sum()):
            raise UnsupportedShapeError(f"observed vector has {bv.size} entries, expected {int((~flags).sum())}")
        b_hat = np.zeros(geo.n)
        b_hat[~flags] = bv
        targets = range(geo.P) if dist_mode else comm.ranks
        for r in targets:
            wb, yb = _y_inputs(geo, flags, b_hat, r)
            if dist_mode and r != me:
                comm.dist.send(torch.from_numpy(wb).to(wire), dst=r, group=comm.group)
                comm.dist.send(torch.from_numpy(yb).to(wire), dst=r, group=comm.group)
            else:
                bits[r], bhat[r] = torch.from_numpy(wb).to(dev), torch.from_numpy(yb).to(dev)
        del b_hat
    else:
        tb = torch.empty((nl + 31) // 32, dtype=torch.int32, device=wire)
        ty = torch.empty(nl, dtype=torch.float64, device=wire)
        comm.dist.recv(tb, src=root, group=comm.group)
        comm.dist.recv(ty, src=root, group=comm.group)
        bits[me], bhat[me] = tb.to(dev), ty.to(dev)
    prob = ShardedProblem(grid, [bits[r] for r in comm.ranks], [bhat[r] for r in comm.ranks])
    lam = config.lam
    if lam is None:  # default_penalty: 0.1 max|A^T Z b_hat| from one residual pass at beta = 0
        zs = [_dev.zeros(nl) for _ in comm.ranks]
        gs = [_dev.empty(nl) for _ in comm.ranks]
        grid.gram(zs, gs, prob.bits_y, prob.bhat_y)
        loc = []
        for g in gs:
            m = ctypes.c_double()
            _lib.call("fl_max_abs", nl, _dev.ptr(g), ctypes.byref(m), _dev.stream())
            loc.append([m.value])
        lam = 0.1 * float(comm.reduce(loc, MAX)[0])
        del zs, gs
        if lam <= 0:
            raise ValueError("penalty must be positive")
    betas, report = sharded_solve(prob, lam, config, observer)
    out = None
    if dist_mode:
        parts = [torch.empty(nl, dtype=torch.float64, device=wire) for _ in range(geo.P)] if me == root else None
        comm.dist.gather(betas[0].contiguous().to(wire), gather_list=parts, dst=root, group=comm.group)
        if me == root:
            out = torch.cat(parts).cpu().numpy()
    else:
        out = geo.from_x([t.cpu().numpy() for t in betas])
    if hasattr(comm, "release_peer_buffers"):
        comm.release_peer_buffers()
    return out, report
