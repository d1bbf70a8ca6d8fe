"""GPU: every instantiated pass-kernel variant agrees with the oracle.

Covers 512-long axes in both layouts (the C4/C5 hot path) and other
power-of-two lengths, for synthesis, analysis and the fused gram, under each
kernel configuration selectable through FL_CFG_STRIDED / FL_CFG_CONTIG
(csrc/fl_fastpass.cu), plus the generic engine (FL_FORCE_GENERIC is read once
per process, so it is exercised in a subprocess).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO
from oracle import fftlasso_oracle as orc

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_2502_04217_b200")

VARIANTS = [10, 5, 7, 12, 15, 2, 4, 28, 31, 36]
# the last two give every persistent CTA several tiles (exercises the
# cross-tile cp.async pipelining)
DIMS = [(512, 4, 8), (4, 6, 512), (16, 512), (512, 2, 64), (2, 512, 16), (512, 128, 64),
        (64, 128, 512)]


def _mask(dims, rng):
    n = int(np.prod(dims))
    return rng.random(n) < 0.15


@pytest.mark.parametrize("var", VARIANTS)
@pytest.mark.parametrize("which", ["FL_CFG_STRIDED", "FL_CFG_CONTIG"])
def test_variant_matches_oracle(var, which, monkeypatch):
    monkeypatch.setenv(which, str(var))
    _check_all_dims(var)


@pytest.mark.parametrize("mode", ["0", "1", "2", "3", "4", "5", "6"])
def test_mirror_engine_matches_oracle(mode, monkeypatch):
    """The mirrored-butterfly engine (FL_MIRROR, m = 64 / 512 / 4096)."""
    monkeypatch.setenv("FL_MIRROR", mode)
    _check_all_dims(int(mode) + 100)
    for dims in [(64, 8, 16), (4096,), (8, 4096), (64, 64, 64), (4096, 4)]:
        _check_dims(dims, np.random.default_rng(len(dims)))


def _check_all_dims(seed):
    rng = np.random.default_rng(seed)
    for dims in DIMS:
        _check_dims(dims, rng)


def _check_dims(dims, rng):
    shape = fl.GridShape(dims)
    flags = _mask(dims, rng)
    mask = fl.Mask.from_bool(flags, shape)
    om = orc.make_mask(dims, flags=flags)
    beta = rng.standard_normal(shape.n)
    x = rng.standard_normal(shape.n)
    tol = 1e-12 * max(1.0, np.abs(beta).max())
    assert np.max(np.abs(fl.synthesize(beta, shape) - orc.synthesize(beta, dims))) <= tol, dims
    assert np.max(np.abs(fl.analyze(x, shape) - orc.analyze(x, dims))) <= tol, dims
    assert np.max(np.abs(fl.gram(beta, mask) - orc.gram(beta, om))) <= tol, dims
    w = rng.standard_normal(mask.n_observed)
    ref = orc.observe_adjoint(w, om)
    assert np.max(np.abs(fl.observe_adjoint(w, mask) - ref)) <= 1e-12 * max(1.0, np.abs(ref).max()), dims


def test_generic_engine_matches_oracle():
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2502_04217_b200 as fl
from oracle import fftlasso_oracle as orc
rng = np.random.default_rng(5)
for dims in [(512, 4, 8), (4, 6, 512), (64, 32), (24, 36), (6, 10, 4)]:
    shape = fl.GridShape(dims)
    flags = rng.random(shape.n) < 0.15
    m, om = fl.Mask.from_bool(flags, shape), orc.make_mask(dims, flags=flags)
    b = rng.standard_normal(shape.n)
    assert np.max(np.abs(fl.synthesize(b, shape) - orc.synthesize(b, dims))) <= 1e-12 * np.abs(b).max(), dims
    assert np.max(np.abs(fl.gram(b, m) - orc.gram(b, om))) <= 1e-12 * np.abs(b).max(), dims
print("ok")
''' % REPO
    env = dict(os.environ, FL_FORCE_GENERIC="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_fused_epilogue_matches_split():
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2502_04217_b200 as fl
from paper_2502_04217_b200 import newton_system as ns
from oracle import fftlasso_oracle as orc
rng = np.random.default_rng(6)
for dims in [(512, 4, 8), (64, 64), (4096,)]:
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
print("ok")
''' % REPO
    env = dict(os.environ, FL_FUSED_EPI="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("split", ["0", "2"])
def test_split_1024_engine_matches_oracle(split):
    """Strided m = 1024 passes with and without the radix-2 split into two
    mirrored 512-point halves (FL_SPLIT is read once per process)."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2502_04217_b200 as fl
from oracle import fftlasso_oracle as orc
rng = np.random.default_rng(11)
for dims in [(1024, 8, 16), (8, 1024, 24), (1024, 1024)]:
    beta = rng.standard_normal(int(np.prod(dims)))
    tol = 1e-12 * np.abs(beta).max()
    sh = fl.GridShape(dims)
    assert np.max(np.abs(fl.synthesize(beta, sh) - orc.synthesize(beta, dims))) <= tol, dims
    assert np.max(np.abs(fl.analyze(beta, sh) - orc.analyze(beta, dims))) <= tol, dims
print("OK")
''' % REPO
    env = dict(os.environ, FL_SPLIT=split)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, out.stderr[-2000:]
