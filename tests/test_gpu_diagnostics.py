"""GPU diagnostics vs the reference (diagnostics.py:112-360, test_diagnostics.py,
test_acceptance.py criterion 3): soft threshold, support sets, the ISTA
oracle on the GPU, and IPM-vs-ISTA objective agreement at sizes the
reference's guarded CPU ISTA refuses.
"""

import json

import numpy as np
import pytest

from conftest import load_golden
from oracle import fftlasso_oracle as orc

pytestmark = pytest.mark.gpu

fl = pytest.importorskip("paper_2502_04217_b200")
from paper_2502_04217_b200 import diagnostics as dg, workloads  # noqa: E402


def test_soft_threshold_bitwise():
    g = load_golden("ista")
    out = dg.soft_threshold(g["soft_x"], float(g["soft_t"]))
    assert out.tobytes() == g["soft_out"].tobytes()
    x = np.array([np.nan, -0.0, 0.0, 0.3, -0.3])
    np.testing.assert_array_equal(np.signbit(dg.soft_threshold(x, 0.3)),
                                  np.signbit(orc.soft_threshold(x, 0.3)))
    assert np.isnan(dg.soft_threshold(x, 0.3)[0])


def test_classify_support():
    c = dg.classify_support(np.zeros(6))
    assert c.n_active == 0 and c.zero.size == 6 and c.threshold == 0.0
    c = dg.classify_support(np.array([1.0, -1.0, 0.0, 0.0]))
    assert c.positive.tolist() == [0] and c.negative.tolist() == [1]
    assert c.active.tolist() == [0, 1]


@pytest.mark.parametrize("name", json.loads(str(load_golden("ista")["cases_json"])))
def test_ista_matches_reference(name):
    g = load_golden("ista")
    dims = tuple(int(d) for d in g[name + "_dims"])
    mask = fl.Mask(g[name + "_missing"], fl.GridShape(dims))
    lam = float(g[name + "_lam"])
    beta, iters = dg.ista_solve(g[name + "_b"], mask, lam, tol=1e-10)
    ref = g[name + "_beta"]
    assert abs(iters - int(g[name + "_iters"])) <= 1
    assert np.max(np.abs(beta - ref)) <= 1e-9 * max(1.0, np.max(np.abs(ref)))
    obj = fl.lasso_objective(beta, g[name + "_b"], mask, lam)
    assert obj == pytest.approx(float(g[name + "_objective"]), rel=1e-12)


def test_ista_empty_mask_fixed_point(rng):
    mask = fl.Mask(np.array([], dtype=np.int64), fl.GridShape((32,)))
    b = rng.standard_normal(32)
    xi = fl.analyze(b, mask.shape)
    beta, iters = dg.ista_solve(b, mask, 0.4, tol=1e-12)
    np.testing.assert_allclose(beta, orc.soft_threshold(xi, 0.4), atol=1e-12)
    assert iters <= 2
    beta0, _ = dg.ista_solve(b, mask, 0.0, tol=1e-12)
    np.testing.assert_allclose(beta0, xi, atol=1e-11)


def test_ista_limits(rng):
    n = 32
    mask = fl.Mask(np.sort(rng.choice(n, 4, replace=False)), fl.GridShape((n,)))
    b = rng.standard_normal(n - 4)
    with pytest.raises(fl.IterationLimitError):
        dg.ista_solve(b, mask, lam=0.3, tol=1e-14, max_iters=3)
    big = fl.Mask(np.array([0]), fl.GridShape((8192,)))
    with pytest.raises(ValueError):
        dg.ista_solve(np.zeros(8191), big, lam=0.1)
    beta, iters = dg.ista_solve(np.zeros(8191), big, lam=0.1, max_n=None)
    assert iters == 1 and not np.any(beta)


def _sparse(rng, n, n_missing, n_active):
    mask = fl.Mask(np.sort(rng.choice(n, n_missing, replace=False)), fl.GridShape((n,)))
    bt = np.zeros(n)
    idx = rng.choice(n, n_active, replace=False)
    bt[idx] = (1.0 + 1.5 * rng.random(n_active)) * np.sign(rng.standard_normal(n_active))
    return fl.observe(bt, mask) + 0.05 * rng.standard_normal(mask.n_observed), mask


def test_acceptance_masked_objectives_agree_with_ista():
    """test_acceptance.py criterion 3 (20 instances) on the GPU: IPM vs ISTA <= 1e-6."""
    worst = 0.0
    for i in range(20):
        rng = np.random.default_rng(3000 + i)
        n = 64 if i % 2 == 0 else 128
        b, mask = _sparse(rng, n, int(round(0.15 * n)), max(2, n // 24))
        beta, rep = fl.solve(b, mask, fl.IpmConfig(lam=0.3, tol=1e-8))
        assert rep.converged
        ref, _ = dg.ista_solve(b, mask, 0.3, tol=1e-10)
        o, o_ref = (fl.lasso_objective(v, b, mask, 0.3) for v in (beta, ref))
        worst = max(worst, abs(o - o_ref) / abs(o_ref))
    assert worst <= 1e-6


@pytest.mark.parametrize("recipe,side", [("c3", 64), ("c4", 64), ("c3", 128)])
def test_ipm_vs_gpu_ista_beyond_cpu_guard(recipe, side):
    """the unguarded GPU ISTA as an independent oracle for
    3D solves far above the reference's n <= 4096 ISTA limit."""
    inst = workloads.c3_bragg(side, seed=0) if recipe == "c3" else workloads.c4_const(side)
    shape = fl.GridShape(inst.dims)
    mask = fl.Mask.from_bool(inst.flags, shape)
    b = fl.observe(inst.beta_true, mask) + inst.noise
    beta, rep = fl.solve(b, mask, fl.IpmConfig(lam=inst.lam, tol=1e-8))
    assert rep.converged
    lam = rep.lam  # the recipe's lambda, or default_penalty when it has none
    ref, iters = dg.ista_solve(b, mask, lam, tol=1e-10, max_iters=20000, max_n=None)
    o, o_ref = (fl.lasso_objective(v, b, mask, lam) for v in (beta, ref))
    assert abs(o - o_ref) <= 1e-6 * abs(o_ref)
    np.testing.assert_array_equal(dg.classify_support(beta).active, dg.classify_support(ref).active)
