"""GPU: every pass-kernel family of the library agrees with the oracle on
multi-tile grids (each persistent CTA / group walks several tiles).

One kernel per (length, layout, kind) -- no run-time switches -- so the
families are reached through the grid shape: the mirrored engine (strided
m = 64 / 512 / 4096), the E = 8 engine (other strided lengths <= 256, all
contiguous lengths outside the group set), the group-decoupled contiguous
passes (m = 512 / 2048, fl_gpass.cuh), the two-stage warp passes (contiguous
m = 1024, fl_wpass.cuh), the mirrored 8 x 16 x 8 engine (strided m = 1024),
the long-fibre E = 16 engine (longer strided fibres), the generic
mixed-radix engine (non-power-of-two even lengths) and the four-step path
(lengths above 8192).
"""

import numpy as np
import pytest

from oracle import fftlasso_oracle as orc

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_2502_04217_b200")
from paper_2502_04217_b200 import _dev, _lib  # noqa: E402
from paper_2502_04217_b200.masking import embed  # noqa: E402

DIMS = [
    # m = 512 both layouts (C4), several tiles per persistent CTA / group
    (512, 4, 8), (4, 6, 512), (16, 512), (512, 2, 64), (2, 512, 16), (512, 128, 64), (64, 128, 512),
    # mirrored m = 64 / 4096 strided, E = 8 lengths, group m = 1024 / 2048 contiguous
    (64, 8, 16), (8, 4096), (4096, 4), (64, 64, 64), (256, 32, 256), (32, 128, 128),
    (4, 1024), (6, 2048), (2, 8, 1024),
    # strided m = 1024 (mirrored 8 x 16 x 8) at small and large strides; strided 2048 (E = 16)
    (1024, 8, 16), (8, 1024, 24), (1024, 1024), (1024, 4, 4096), (2048, 4, 8),
    # generic mixed-radix and four-step
    (24, 36), (6, 10, 4), (96, 40, 24), (16384,), (2, 16384),
]


@pytest.mark.parametrize("dims", DIMS)
def test_pass_families_match_oracle(dims):
    rng = np.random.default_rng(sum(dims))
    shape = fl.GridShape(dims)
    flags = rng.random(shape.n) < 0.15
    mask = fl.Mask.from_bool(flags, shape)
    om = orc.make_mask(dims, flags=flags)
    beta = rng.standard_normal(shape.n)
    x = rng.standard_normal(shape.n)
    tol = 1e-12 * max(1.0, np.abs(beta).max())
    assert np.max(np.abs(fl.synthesize(beta, shape) - orc.synthesize(beta, dims))) <= tol
    assert np.max(np.abs(fl.analyze(x, shape) - orc.analyze(x, dims))) <= tol
    assert np.max(np.abs(fl.gram(beta, mask) - orc.gram(beta, om))) <= tol
    w = rng.standard_normal(mask.n_observed)
    ref = orc.observe_adjoint(w, om)
    assert np.max(np.abs(fl.observe_adjoint(w, mask) - ref)) <= 1e-12 * max(1.0, np.abs(ref).max())
    # residual pass A^T Z (b_hat - A beta), the solver's data correlation
    ref_r = orc.observe_adjoint(w - orc.observe(beta, om), om)
    bh = _dev.to_dev(embed(w, mask))
    bd = _dev.to_dev(beta)
    g = _dev.empty(shape.n)
    _lib.call("fl_residual_adjoint", _dev.plan_for(dims).handle, _dev.ptr(mask.on_device().bits), _dev.ptr(bh),
              _dev.ptr(bd), _dev.ptr(g), _dev.stream())
    assert np.max(np.abs(g.cpu().numpy() - ref_r)) <= 1e-12 * max(1.0, np.abs(ref_r).max())


def test_kkt_apply_epilogue_families(rng):
    """KKT epilogue: separate 16-byte pass (2D/3D) and fused into the
    contiguous gram pass (1D, group and E = 8 engines)."""
    from paper_2502_04217_b200 import newton_system as ns

    for dims in [(512, 4, 8), (64, 64), (4096,), (512,), (1024,), (96,)]:
        shape = fl.GridShape(dims)
        flags = rng.random(shape.n) < 0.15
        m, om = fl.Mask.from_bool(flags, shape), orc.make_mask(dims, flags=flags)
        s = [rng.random(shape.n) + 0.4 for _ in range(4)]
        d, od = ns.barrier_diagonals(*s), orc.diagonals(*s)
        db, dz = rng.standard_normal(shape.n), rng.standard_normal(shape.n)
        t, b = ns.apply_kkt(db, dz, d, m)
        ot, ob = orc.kkt_apply(db, dz, od, om)
        assert np.max(np.abs(t - ot)) <= 1e-11, dims
        assert np.array_equal(b, ob), dims
