"""Test-only CPU backend of sharded.ShardOps: the oracle's per-axis transforms
and NumPy reshapes for the slab transposes.  It exercises the sharded
orchestration (layouts, all-to-all plumbing, reductions) on CPU with gloo;
the CUDA kernels implementing the same interface are tested on the GPU.
"""

import numpy as np
import torch

from oracle import fftlasso_oracle as orc


class NumpyShardOps:
    def __init__(self, geo):
        self.geo = geo

    @staticmethod
    def empty(n):
        return torch.empty(int(n), dtype=torch.float64)

    @staticmethod
    def vec(a):
        return torch.from_numpy(np.array(a, dtype=np.float64).reshape(-1))

    @staticmethod
    def bits(flags):
        return torch.from_numpy(np.array(flags, dtype=bool).reshape(-1))

    def _x(self, t):
        g = self.geo
        return t.numpy().reshape(g.a, g.dims[1], g.dims[2])

    def _y(self, t):
        g = self.geo
        return t.numpy().reshape(g.b, g.dims[2], g.dims[0])

    def synth_x(self, src, dst):
        x = orc.synth_axis(orc.synth_axis(self._x(src), 2), 1)
        dst.copy_(torch.from_numpy(np.ascontiguousarray(x).reshape(-1)))

    def analyze_x(self, src, dst):
        x = orc.analyze_axis(orc.analyze_axis(self._x(src), 1), 2)
        dst.copy_(torch.from_numpy(np.ascontiguousarray(x).reshape(-1)))

    def synth_y0(self, src, dst):
        y = orc.synth_axis(self._y(src), 2)
        dst.copy_(torch.from_numpy(np.ascontiguousarray(y).reshape(-1)))

    def fused_y(self, bits, bhat, src, dst, want_norm):
        y = orc.synth_axis(self._y(src), 2).reshape(-1).copy()
        miss = bits.numpy()
        if bhat is None:
            y[miss] = 0.0
        else:
            y = np.where(miss, 0.0, bhat.numpy() - y)
        nrm = float(y @ y)
        g = self.geo
        out = orc.analyze_axis(y.reshape(g.b, g.dims[2], g.dims[0]), 2)
        dst.copy_(torch.from_numpy(np.ascontiguousarray(out).reshape(-1)))
        return nrm

    def pack_x(self, x, send):
        g = self.geo
        blocks = self._x(x).reshape(g.a, g.P, g.b, g.dims[2]).transpose(1, 0, 2, 3)
        send.copy_(torch.from_numpy(np.ascontiguousarray(blocks).reshape(-1)))

    def unpack_y(self, recv, y):
        g = self.geo
        blocks = recv.numpy().reshape(g.P, g.a, g.b, g.dims[2])
        y.copy_(torch.from_numpy(np.ascontiguousarray(blocks.transpose(2, 3, 0, 1)).reshape(-1)))

    def pack_y(self, y, send):
        g = self.geo
        blocks = self._y(y).reshape(g.b, g.dims[2], g.P, g.a).transpose(2, 3, 0, 1)
        send.copy_(torch.from_numpy(np.ascontiguousarray(blocks).reshape(-1)))

    def unpack_x(self, recv, x):
        g = self.geo
        blocks = recv.numpy().reshape(g.P, g.a, g.b, g.dims[2])
        x.copy_(torch.from_numpy(np.ascontiguousarray(blocks.transpose(1, 0, 2, 3)).reshape(-1)))

    # peer exchange: write straight into the owning rank's slab (``table`` holds
    # every rank's buffer as a NumPy array; see ShmPeerComm)
    def x_to_y_peers(self, rank, x, table):
        g = self.geo
        xs = self._x(x)  # (a, d1, d2)
        for r2, buf in enumerate(table):
            y = buf.reshape(g.b, g.dims[2], g.dims[0])
            y[:, :, rank * g.a:(rank + 1) * g.a] = xs[:, r2 * g.b:(r2 + 1) * g.b, :].transpose(1, 2, 0)

    def y_to_x_peers(self, rank, y, table):
        g = self.geo
        ys = self._y(y)  # (b, d2, d0)
        for r2, buf in enumerate(table):
            xr = buf.reshape(g.a, g.dims[1], g.dims[2])
            xr[:, rank * g.b:(rank + 1) * g.b, :] = ys[:, :, r2 * g.a:(r2 + 1) * g.a].transpose(2, 0, 1)


class ShmPeerComm:
    """CPU stand-in for the CUDA-IPC peer buffers of sharded.DistComm: POSIX
    shared memory created by each rank, names all-gathered over gloo, every
    rank maps every buffer; the barrier is a gloo barrier.  Everything else
    is DistComm's."""

    def __new__(cls, *a, **k):
        from paper_2502_04217_b200.sharded import DistComm

        class _Shm(DistComm):
            def peer_buffers(self, n):
                from multiprocessing import shared_memory

                mine = shared_memory.SharedMemory(create=True, size=int(n) * 8)
                names = [None] * self.world
                self.dist.all_gather_object(names, mine.name)
                maps = [mine if nm == mine.name else shared_memory.SharedMemory(name=nm) for nm in names]
                self._shm = getattr(self, "_shm", []) + [(mine, maps)]
                arrays = [np.ndarray((int(n),), dtype=np.float64, buffer=m.buf) for m in maps]
                return [torch.from_numpy(arrays[self.ranks[0]])], [arrays]

            def barrier(self):
                self.dist.barrier()

            def close(self):
                self.dist.barrier()
                for mine, maps in getattr(self, "_shm", []):
                    for m in maps:
                        if m is not mine:
                            m.close()
                    mine.close()
                    mine.unlink()
                self._shm = []

        return _Shm(*a, **k)
