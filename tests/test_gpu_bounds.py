"""GPU: out-of-bounds write detection with guard regions (compute-sanitizer is
closed on this GPU pool, so memory safety is checked with our own canaries).

Every output of every pass family is written into the middle of a larger
buffer whose head and tail hold a NaN-payload canary; after the call the
canaries must be bit-identical and the result must still match the oracle.
Inputs sit between canaries too, so a kernel that reads past its input would
pull a NaN into the result (caught by the oracle comparison).
"""

import ctypes

import numpy as np
import pytest

from oracle import fftlasso_oracle as orc

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_2502_04217_b200")
import torch  # noqa: E402

from paper_2502_04217_b200 import _dev, _lib  # noqa: E402
from paper_2502_04217_b200 import sharded as sh  # noqa: E402

PAD = 4096  # doubles on each side (32 KiB)
CANARY = np.frombuffer(np.uint64(0x7FF8DEADBEEF1234).tobytes(), dtype=np.float64)[0]


def guarded(values=None, n=None):
    n = len(values) if values is not None else n
    buf = torch.full((n + 2 * PAD,), float(CANARY), dtype=torch.float64, device="cuda")
    buf.view(torch.int64).fill_(0x7FF8DEADBEEF1234)
    if values is not None:
        buf[PAD:PAD + n] = torch.from_numpy(np.asarray(values, dtype=np.float64)).cuda()
    return buf, buf[PAD:PAD + n]


def intact(buf, n):
    raw = buf.view(torch.int64).cpu().numpy()
    return bool(np.all(raw[:PAD] == 0x7FF8DEADBEEF1234) and np.all(raw[PAD + n:] == 0x7FF8DEADBEEF1234))


DIMS = [(512, 4, 8), (4, 6, 512), (2, 8, 1024), (1024, 4, 4096), (8, 1024, 24), (64, 64, 64), (96, 40, 24),
        (4096,), (16384,), (24, 36)]


@pytest.mark.parametrize("dims", DIMS)
def test_pass_families_stay_in_bounds(dims):
    rng = np.random.default_rng(len(dims) + dims[0])
    shape = fl.GridShape(dims)
    n = shape.n
    plan = _dev.plan_for(dims)
    flags = rng.random(n) < 0.15
    mask = fl.Mask.from_bool(flags, shape)
    om = orc.make_mask(dims, flags=flags)
    bits = mask.on_device().bits
    beta = rng.standard_normal(n)
    ibuf, inp = guarded(beta)
    tol = 1e-12 * np.abs(beta).max()
    for name, call, ref in [
        ("synthesize", lambda o: _lib.call("fl_synthesize", plan.handle, _dev.ptr(inp), _dev.ptr(o), _dev.stream()),
         orc.synthesize(beta, dims)),
        ("analyze", lambda o: _lib.call("fl_analyze", plan.handle, _dev.ptr(inp), _dev.ptr(o), _dev.stream()),
         orc.analyze(beta, dims)),
        ("gram", lambda o: _lib.call("fl_gram", plan.handle, _dev.ptr(bits), _dev.ptr(inp), _dev.ptr(o),
                                     _dev.stream()), orc.gram(beta, om)),
    ]:
        obuf, out = guarded(n=n)
        call(out)
        torch.cuda.synchronize()
        assert intact(obuf, n), (name, dims)
        assert intact(ibuf, n), (name, dims)
        assert np.max(np.abs(out.cpu().numpy() - ref)) <= tol, (name, dims)


def test_kkt_and_exchange_stay_in_bounds():
    rng = np.random.default_rng(9)
    dims = (64, 32, 512)
    shape = fl.GridShape(dims)
    n = shape.n
    flags = rng.random(n) < 0.15
    mask = fl.Mask.from_bool(flags, shape)
    s = [rng.random(n) + 0.4 for _ in range(4)]
    sig = [guarded(x / y) for x, y in ((s[2], s[0]), (s[3], s[1]))]
    db, dz = rng.standard_normal(n), rng.standard_normal(n)
    (bb, bv), (zb, zv) = guarded(db), guarded(dz)
    (tb, tv), (ob, ov) = guarded(n=n), guarded(n=n)
    pkp = ctypes.c_double()
    _lib.call("fl_kkt_apply", _dev.plan_for(dims).handle, _dev.ptr(mask.on_device().bits), _dev.ptr(sig[0][1]),
              _dev.ptr(sig[1][1]), _dev.ptr(bv), _dev.ptr(zv), _dev.ptr(tv), _dev.ptr(ov), ctypes.byref(pkp),
              _dev.stream())
    torch.cuda.synchronize()
    assert all(intact(b, n) for b in (bb, zb, tb, ob, sig[0][0], sig[1][0]))
    od = orc.diagonals(*s)
    ot, obot = orc.kkt_apply(db, dz, od, orc.make_mask(dims, flags=flags))
    assert np.max(np.abs(tv.cpu().numpy() - ot)) <= 1e-11 and np.array_equal(ov.cpu().numpy(), obot)
    # slab exchange (peer kernels) into guarded receive slabs, 4 emulated ranks
    P = 4
    geo = sh.SlabGeometry(dims, P)
    nl = geo.n_local
    x = rng.standard_normal(n)
    recv = [guarded(n=nl) for _ in range(P)]
    table = (ctypes.c_void_p * P)(*(v.data_ptr() for _, v in recv))
    xs = [guarded(geo.x_slab(x, r)) for r in range(P)]
    for r in range(P):
        _lib.call("fl_slab_x_to_y_peers", geo.a, dims[1], dims[2], P, r, _dev.ptr(xs[r][1]),
                  ctypes.cast(table, ctypes.POINTER(ctypes.c_void_p)), _dev.stream())
    torch.cuda.synchronize()
    for r in range(P):
        assert intact(recv[r][0], nl) and intact(xs[r][0], nl)
        assert recv[r][1].cpu().numpy().tobytes() == geo.y_slab(x, r).tobytes()
