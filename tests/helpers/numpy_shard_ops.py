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
