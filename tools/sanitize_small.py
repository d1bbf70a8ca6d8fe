"""Small operator + solve calls hitting every kernel family (for compute-sanitizer).

Covers the E=8 register engine (strided and contiguous, every pass kind), the
mirrored engine (m = 64 / 512), the generic mixed-radix engine, the four-step
long-axis path, the slab transposes and a short IPM solve.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from paper_2502_04217_b200 import sharded as sh  # noqa: E402

rng = np.random.default_rng(3)
for dims in [(16, 8, 32), (64, 16, 16), (512, 2, 4), (4, 2, 512), (6, 10, 12), (16384,), (24, 36)]:
    g = fl.GridShape(dims)
    m = fl.Mask.from_bool(rng.random(g.n) < 0.2, g)
    b = rng.standard_normal(g.n)
    fl.synthesize(b, g)
    fl.analyze(b, g)
    fl.gram(b, m)
    fl.observe_adjoint(rng.standard_normal(m.n_observed), m)
grid = sh.ShardedGrid((8, 8, 16), sh.LocalComm(2))
xs = [fl._dev.to_dev(rng.standard_normal(grid.geo.n_local)) for _ in range(2)]
ys = [fl._dev.empty(grid.geo.n_local) for _ in range(2)]
grid.synthesize_to_y(xs, ys)
g = fl.GridShape((32,))
m = fl.Mask.from_bool(rng.random(32) < 0.2, g)
beta, rep = fl.solve(rng.standard_normal(m.n_observed), m, fl.IpmConfig(lam=0.3, max_iters=3))
print("ok", rep.iterations)
