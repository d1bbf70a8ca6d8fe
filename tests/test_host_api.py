"""CPU: host-side logic of the drop-in API (validation, packing, configs, errors).

Mirrors the reference's validation tests (test_fourier.py:22-90,
test_masking.py:25-54, test_pcg.py:31-43, test_ipm.py config/schedule).
"""

import numpy as np
import pytest

import paper_2502_04217_b200 as fl
from paper_2502_04217_b200 import ipm
from paper_2502_04217_b200.pcg import PcgConfig
from oracle import fftlasso_oracle as orc


class TestGridShape:
    def test_valid(self):
        g = fl.GridShape((4, 6, 8))
        assert g.n == 192 and g.ndim == 3

    @pytest.mark.parametrize("dims", [(5,), (4, 7), (3, 3, 3), (0,), (2, 2, 2, 2), ()])
    def test_rejects_bad_dims(self, dims):
        with pytest.raises(fl.UnsupportedShapeError):
            fl.GridShape(dims)


class TestPackUnpack:
    def test_known_values(self):
        beta = fl.pack(0.5 * np.ones(4, dtype=complex), fl.GridShape((4,)))
        np.testing.assert_allclose(beta, [0.5, 0.5, 0.70710678, 0.0], atol=1e-8)
        v = np.array([5.0, -1.0 + 1.0j, -1.0, -1.0 - 1.0j])
        np.testing.assert_allclose(fl.pack(v, fl.GridShape((4,))), [5.0, -1.0, -1.41421356, 1.41421356],
                                   atol=1e-8)
        np.testing.assert_allclose(fl.unpack(np.array([5.0, -1.0, -np.sqrt(2), np.sqrt(2)]),
                                             fl.GridShape((4,))), v, atol=1e-12)

    @pytest.mark.parametrize("dims", [(32,), (4, 6, 4), (10, 6)])
    def test_mutual_inverse(self, dims, rng):
        g = fl.GridShape(dims)
        beta = rng.standard_normal(g.n)
        np.testing.assert_allclose(fl.pack(fl.unpack(beta, g), g), beta, rtol=0, atol=1e-15)

    def test_unpack_is_the_spectrum_of_synthesis(self, rng):
        """unpack(beta) == ortho DFT of synthesize(beta) (oracle as the checker)."""
        dims = (6, 4, 8)
        beta = rng.standard_normal(int(np.prod(dims)))
        x = orc.synthesize(beta, dims).reshape(dims)
        np.testing.assert_allclose(fl.unpack(beta, fl.GridShape(dims)),
                                   np.fft.fftn(x, norm="ortho").reshape(-1), atol=1e-12)

    def test_rejects_asymmetric(self):
        with pytest.raises(fl.MalformedSpectrumError):
            fl.pack(np.array([1.0, 2.0 + 1.0j, 0.0, 99.0]), fl.GridShape((4,)))
        with pytest.raises(fl.UnsupportedShapeError):
            fl.pack(np.zeros(5, dtype=complex), fl.GridShape((4,)))


class TestMask:
    def test_basic(self):
        m = fl.Mask(np.array([1, 5]), fl.GridShape((8,)))
        assert m.n_missing == 2 and m.n_observed == 6 and m.missing_bool.sum() == 2

    def test_validation(self):
        g = fl.GridShape((8,))
        for bad in ([8], [-1], [3, 3], [5, 2], list(range(8))):
            with pytest.raises(ValueError):
                fl.Mask(np.array(bad), g)
        np.testing.assert_array_equal(fl.Mask.from_bool([0, 1, 0, 0, 1, 0, 0, 0], g).missing, [1, 4])
        with pytest.raises(fl.UnsupportedShapeError):
            fl.Mask.from_bool([0, 1], g)


class TestConfigs:
    @pytest.mark.parametrize("kwargs", [{"sigma_mu": 0.0}, {"sigma_mu": 1.0}, {"ftb_tau": 1.0},
                                        {"tol": 0.0}])
    def test_ipm_rejects_bad_parameters(self, kwargs):
        with pytest.raises(ValueError):
            fl.IpmConfig(**kwargs)

    def test_pcg_config(self):
        with pytest.raises(ValueError):
            PcgConfig(abs_tol=0.0, rel_tol=0.0)
        with pytest.raises(ValueError):
            PcgConfig(abs_tol=-1.0)
        assert PcgConfig().iteration_limit(10) == 100
        assert PcgConfig().iteration_limit(10 ** 6) == 5000
        assert PcgConfig(max_iters=7).iteration_limit(10 ** 6) == 7

    def test_barrier_schedule(self):
        cfg = fl.IpmConfig(tol=1e-8)
        assert ipm.next_barrier(1.0, cfg.tol, cfg) == pytest.approx(0.2)
        assert ipm.next_barrier(1e-4, cfg.tol, cfg) == pytest.approx(1e-6)
        assert ipm.next_barrier(1e-9, cfg.tol, cfg) == pytest.approx(1e-9)

    def test_alpha_from_ratio(self):
        assert ipm._alpha_from_ratio(float("inf"), 0.995) == 1.0
        assert ipm._alpha_from_ratio(0.5, 0.995) == pytest.approx(0.995 * 0.5)
        assert ipm._alpha_from_ratio(3.0, 0.995) == 1.0


def test_no_cpu_fallback():
    """Without a CUDA device every numeric entry point fails loudly."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = fl.GridShape((8,))
    with pytest.raises(fl.BackendUnavailableError):
        fl.synthesize(np.zeros(8), g)
    with pytest.raises(fl.BackendUnavailableError):
        fl.solve(np.zeros(8), fl.Mask(np.array([], dtype=np.int64), g))


def test_report_schema_keys():
    rec = ipm.IterationRecord(1, 0.1, 0.0, 0.0, 0.0, 0.0, 3, 1.0, 1.0, 0.0, True, 0.0)
    assert list(rec.to_dict()) == ["record", "iteration", "mu", "primal_inf", "dual_inf",
                                   "complementarity", "kkt_max", "krylov_iters", "alpha_primal",
                                   "alpha_dual", "pcg_residual", "centrality_ok", "wall_time"]


def _verdict(status, k=3, norm=1e-9, bad=0.0, ap=0.5, ad=0.25, skip=0.0, interior=0.0):
    import torch

    v = torch.zeros(16, dtype=torch.float64)
    v[4], v[5], v[6], v[7] = ap, ad, skip, interior
    v[8], v[9], v[10], v[11], v[12] = status, k, norm, bad, 1.0
    return type("WS", (), {"verdict": v, "x": None})()


def test_step_verdict_maps_device_statuses_to_reference_errors():
    """Host side of the one-sync IPM step (ipm._step_verdict): the device
    verdict raises what the synchronous path raises, in the same order."""
    res, ap, ad = ipm._step_verdict(_verdict(1))
    assert (res.iterations, res.converged, ap, ad) == (3, True, 0.5, 0.25)
    with pytest.raises(fl.InteriorViolationError):
        ipm._step_verdict(_verdict(5, skip=1.0))
    with pytest.raises(fl.NumericalBreakdownError, match="curvature"):
        ipm._step_verdict(_verdict(3, bad=-1.0, skip=1.0))
    with pytest.raises(fl.NumericalBreakdownError, match="preconditioner produced"):
        ipm._step_verdict(_verdict(4, k=0, bad=float("nan"), skip=1.0))
    with pytest.raises(fl.NumericalBreakdownError, match="at iteration 7"):
        ipm._step_verdict(_verdict(4, k=7, bad=-2.0, skip=1.0))
    with pytest.raises(fl.NumericalBreakdownError, match="PCG stalled"):
        ipm._step_verdict(_verdict(2, skip=1.0))
    with pytest.raises(fl.StalledError, match="collapsed"):
        ipm._step_verdict(_verdict(1, ap=1e-13, skip=1.0))
    with pytest.raises(fl.StalledError, match="interior"):
        ipm._step_verdict(_verdict(1, interior=1.0))
