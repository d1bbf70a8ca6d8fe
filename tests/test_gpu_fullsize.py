"""GPU parity at BASELINE's full sizes through size-independent properties.

The CPU oracle cannot run at C4 (512^3) / C5 (1024^3) sizes in the test
budget, so the operators are checked on the device with exact algebraic
identities of the reference's operators (fourier.py:14-16, masking.py:107-118,
newton_system.py:148-152):

* A is orthogonal: analyze(synthesize(x)) = x and ||A x|| = ||x||;
* G = A^T Z A is a symmetric orthogonal projector: u.Gv = v.Gu, G(Gu) = Gu;
* the condensed KKT matrix is symmetric: d1.K d2 = d2.K d1;
* the slab-sharded gram (C5 layout, P = 8 ranks emulated in one process)
  equals the single-GPU gram.

Bragg-punched masks (15.1 % missing) as in the C3-C5 recipes.  Everything
stays on the device (torch only for the random inputs and the dot products).
"""

from types import SimpleNamespace

import pytest

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_2502_04217_b200")
torch = pytest.importorskip("torch")
from paper_2502_04217_b200 import newton_system as ns, sharded as sh, workloads  # noqa: E402


def _rand(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(n, dtype=torch.float64, device="cuda", generator=g)


def _rel_max(a, b):
    return float((a - b).abs().max() / b.abs().max())


@pytest.fixture(scope="module", params=[512, 1024], ids=["C4-512^3", "C5-1024^3"])
def grid(request):
    side = request.param
    shape = fl.GridShape((side,) * 3)
    mask = fl.Mask.from_bool(workloads.bragg_flags(side), shape)
    mask.on_device()
    yield side, shape, mask
    torch.cuda.empty_cache()


def test_transform_orthogonal(grid):
    side, shape, _ = grid
    x = _rand(shape.n, 1)
    y = fl.synthesize(x, shape)
    assert abs(float(torch.linalg.vector_norm(y) / torch.linalg.vector_norm(x)) - 1.0) <= 1e-12
    z = fl.analyze(y, shape)
    del y
    assert _rel_max(z, x) <= 1e-12


def test_gram_symmetric_projector(grid):
    side, shape, mask = grid
    u, v = _rand(shape.n, 2), _rand(shape.n, 3)
    gu = fl.gram(u, mask)
    gv = fl.gram(v, mask)
    a, b = float(u @ gv), float(v @ gu)
    assert abs(a - b) <= 1e-11 * abs(a)
    del gv
    ggu = fl.gram(gu, mask)
    assert _rel_max(ggu, gu) <= 1e-12
    del ggu
    # ||Z A u||^2 = u.Gu, and u.Gu <= ||u||^2
    assert float(u @ gu) <= float(u @ u)


def test_kkt_symmetric(grid):
    side, shape, mask = grid
    n = shape.n
    # apply_kkt reads only sigma1, sigma2 (the other diagonals are derived)
    d = SimpleNamespace(sigma1=_rand(n, 10).abs() + 0.4, sigma2=_rand(n, 11).abs() + 0.4)
    d1b, d1z, d2b, d2z = (_rand(n, 20 + i) for i in range(4))
    t1, b1 = ns.apply_kkt(d1b, d1z, d, mask)
    t2, b2 = ns.apply_kkt(d2b, d2z, d, mask)
    lhs = float(d2b @ t1 + d2z @ b1)
    rhs = float(d1b @ t2 + d1z @ b2)
    assert abs(lhs - rhs) <= 1e-11 * abs(lhs)


def test_sharded_gram_c5_layout_matches_single_gpu(grid):
    side, shape, mask = grid
    P = 8
    comm = sh.LocalComm(P)
    sg = sh.ShardedGrid(shape.dims, comm)
    geo = sg.geo
    bits = [sg.ops[0].bits(sh.bragg_y_flags(geo, r)) for r in comm.ranks]
    u = _rand(shape.n, 4)
    ref = fl.gram(u, mask)
    nl = geo.n_local
    xs = [u[r * nl:(r + 1) * nl] for r in comm.ranks]
    out = [fl._dev.empty(nl) for _ in comm.ranks]
    sg.gram(xs, out, bits, want_norm=False)
    got = torch.cat(out)
    del out, xs
    assert _rel_max(got, ref) <= 1e-12


def test_kkt_apply_operator_order(grid):
    """fl_kkt_apply's operator order (fl_kkt_order): at 512^3 order B (the
    contiguous axis first and last, the fused mask pass on axis 0, the KKT
    epilogue fused into the final analysis), at 1024^3 order A.  Either way
    the result equals the gram (order A, fl_gram) followed by the separate
    epilogue pass: top to rounding, bottom bitwise (it does not depend on the
    gram), d.Kd to rounding."""
    import ctypes

    from paper_2502_04217_b200 import _dev, _lib

    side, shape, mask = grid
    n = shape.n
    plan = _dev.plan_for(shape.dims)
    assert _lib.lib().fl_kkt_order(plan.handle) == (1 if side == 512 else 0)
    s1, s2 = _rand(n, 30).abs() + 0.4, _rand(n, 31).abs() + 0.4
    db, dz = _rand(n, 32), _rand(n, 33)
    bits = mask.on_device().bits
    top, bot, pkp = _dev.empty(n), _dev.empty(n), ctypes.c_double()
    _lib.call("fl_kkt_apply", plan.handle, _dev.ptr(bits), _dev.ptr(s1), _dev.ptr(s2), _dev.ptr(db),
              _dev.ptr(dz), _dev.ptr(top), _dev.ptr(bot), ctypes.byref(pkp), _dev.stream())
    g = fl.gram(db, mask)
    bot2, pkp2 = _dev.empty(n), ctypes.c_double()
    _lib.call("fl_kkt_epilogue", n, _dev.ptr(g), _dev.ptr(db), _dev.ptr(dz), _dev.ptr(s1), _dev.ptr(s2),
              _dev.ptr(bot2), ctypes.byref(pkp2), _dev.stream())
    assert _rel_max(top, g) <= 1e-12
    assert torch.equal(bot, bot2)
    assert abs(pkp.value - pkp2.value) <= 1e-12 * abs(pkp2.value)
