"""CPU: the oracle restatement reproduces the reference's golden vectors.

The fixtures in tests/golden were recorded from the real reference package by
oracle/make_golden.py; this pins the oracle before any GPU test trusts it.
"""

import json

import numpy as np
import pytest

from conftest import load_golden
from oracle import fftlasso_oracle as orc


def test_transforms_match_reference_and_trig_formula():
    g = load_golden("transforms")
    for dims in json.loads(str(g["dims_json"])):
        key = "x".join(map(str, dims))
        np.testing.assert_array_equal(orc.synthesize(g[key + "__beta"], dims), g[key + "__synth"])
        np.testing.assert_array_equal(orc.analyze(g[key + "__x"], dims), g[key + "__analyze"])
        n = int(np.prod(dims))
        if n <= 1024:
            a = orc.dense_synthesis(dims)
            assert np.max(np.abs(a @ g[key + "__beta"] - g[key + "__synth"])) <= 1e-12
            assert np.max(np.abs(a.T @ g[key + "__x"] - g[key + "__analyze"])) <= 1e-12


def test_masking_matches_reference():
    g = load_golden("masking")
    for dims, _ in json.loads(str(g["cases_json"])):
        key = "x".join(map(str, dims))
        m = orc.make_mask(dims, missing=g[key + "__missing"])
        np.testing.assert_array_equal(orc.observe(g[key + "__beta"], m), g[key + "__observe"])
        np.testing.assert_array_equal(orc.embed(g[key + "__vals"], m), g[key + "__embed"])
        np.testing.assert_array_equal(orc.observe_adjoint(g[key + "__vals"], m), g[key + "__adjoint"])
        np.testing.assert_array_equal(orc.gram(g[key + "__beta"], m), g[key + "__gram"])


def _state(g, key):
    return orc.OState(**{f: g[f"{key}__st_{f}"].copy() for f in
                         ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2")},
                      mu=float(g[key + "__mu"]))


def test_newton_system_matches_reference_bitwise():
    g = load_golden("newton")
    for dims, _ in json.loads(str(g["cases_json"])):
        key = "x".join(map(str, dims))
        m = orc.make_mask(dims, missing=g[key + "__missing"])
        st = _state(g, key)
        d = orc.diagonals(st.s1, st.s2, st.nu1, st.nu2)
        for i, f in enumerate(("sigma1", "sigma2", "lambda1", "lambda2", "dvec", "bvec")):
            np.testing.assert_array_equal(d[i], g[f"{key}__diag_{f}"])
        rhs = orc.newton_rhs(st, g[key + "__b"], m, float(g[key + "__lam"]))
        for f in ("r1", "r2", "r3", "r4", "r5", "r6", "r_beta", "r_c"):
            np.testing.assert_array_equal(rhs[f], g[f"{key}__rhs_{f}"])
        top, bot = orc.kkt_apply(g[key + "__db"], g[key + "__dz"], d, m)
        np.testing.assert_array_equal(top, g[key + "__kkt_top"])
        np.testing.assert_array_equal(bot, g[key + "__kkt_bottom"])
        pt, pb = orc.precond_apply(g[key + "__db"], g[key + "__dz"], d)
        np.testing.assert_array_equal(pt, g[key + "__pinv_top"])
        np.testing.assert_array_equal(pb, g[key + "__pinv_bottom"])
        rec = orc.recover(g[key + "__db"], g[key + "__dz"], rhs, d)
        for i, f in enumerate(("d_s1", "d_s2", "d_y1", "d_y2")):
            np.testing.assert_array_equal(rec[i], g[f"{key}__rec_{f}"])


@pytest.mark.parametrize("name", ["c1_4096", "c4_32", "harm_8", "empty_128", "maxit_64"])
def test_solve_trajectories_match_reference(name):
    g = load_golden("solve_" + name)
    dims = tuple(int(d) for d in g["dims"])
    m = orc.make_mask(dims, missing=g["missing"])
    lam = float(g["lam"])
    recs = json.loads(str(g["records_json"]))
    cfg = orc.OConfig(lam=lam, tol=1e-8, max_iters=3 if name == "maxit_64" else 200)
    beta, rep = orc.solve(g["b"], m, cfg)
    assert rep.status == str(g["status"])
    assert rep.krylov_counts == [r["krylov_iters"] for r in recs]
    np.testing.assert_allclose(beta, g["beta"], rtol=0, atol=1e-15 * max(1.0, np.abs(g["beta"]).max()))
    assert abs(rep.final_objective - float(g["final_objective"])) <= 1e-14 * abs(float(g["final_objective"]))


def test_ista_and_soft_threshold_match_reference():
    g = load_golden("ista")
    out = orc.soft_threshold(g["soft_x"], float(g["soft_t"]))
    assert out.tobytes() == g["soft_out"].tobytes()
    for name in json.loads(str(g["cases_json"])):
        m = orc.make_mask(tuple(g[name + "_dims"]), missing=g[name + "_missing"])
        beta, iters = orc.ista(g[name + "_b"], m, float(g[name + "_lam"]), tol=1e-10)
        assert iters == int(g[name + "_iters"])
        np.testing.assert_array_equal(beta, g[name + "_beta"])
        assert orc.lasso_objective(beta, g[name + "_b"], m, float(g[name + "_lam"])) == \
            float(g[name + "_objective"])


def test_dense_spectrum_probe_matches_reference():
    """oracle.dense_condensed / preconditioned_spectrum == reference
    diagnostics.py:94-224 on two observer snapshots of a reference solve."""
    g = load_golden("spectrum")
    m = orc.make_mask((24,), missing=g["missing"])
    fields = ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2")
    for tag in ("first", "last"):
        st = orc.OState(*(g[f"{tag}__{f}"] for f in fields), mu=0.0)
        k, p = orc.dense_condensed(st, m)
        assert k.tobytes() == g[f"{tag}__K"].tobytes() and p.tobytes() == g[f"{tag}__P"].tobytes()
        rep = orc.preconditioned_spectrum(st, m)
        np.testing.assert_array_equal(rep["eigenvalues"], g[f"{tag}__eigs"])
        sc = g[f"{tag}__scalars"]
        got = [rep["unit_cluster_size"], rep["predicted_cluster_size"], rep["kappa_observed"], rep["kappa_predicted"],
               rep["kappa_unpreconditioned"], rep["n_active"], rep["strict_complementarity"], rep["duality_measure"]]
        np.testing.assert_array_equal(np.array(got, dtype=np.float64), sc)
