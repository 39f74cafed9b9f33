"""Host side of the batched Monte-Carlo harness (simulate.py) against the reference's own
outputs (tests/golden/mc_small.npz, made by tests/golden/make_mc_golden.py): geometry and every
synthesized realization bit-exact, Wilson intervals, CSV contract, validation."""

import os

import numpy as np
import pytest

from paper_1805_01759_b200 import simulate as S
from paper_1805_01759_b200.exceptions import ConfigurationError, GeometryError
from paper_1805_01759_b200.geometry import AcquisitionGeometry, steering_column
from paper_1805_01759_b200.solver import SolverConfig

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def mc():
    return np.load(os.path.join(HERE, "golden", "mc_small.npz"))


def test_demo_geometry_bit_exact(mc):
    g = S.demo_geometry()
    assert np.array_equal(g.baselines, mc["baselines"])
    assert np.array_equal(g.times, mc["times"])


@pytest.mark.parametrize("tag,dphi", [("phi0", 0.0), ("phirand", None)])
def test_realizations_bit_exact(mc, tag, dphi):
    base = S.Scenario(geometry=S.demo_geometry(), seed=int(mc["seed"]))
    setup = S.MonteCarloSetup(delta_phi=dphi, solver=SolverConfig(max_iters=300, tol=1e-6))
    grid = S.harness_grid(base, setup)
    r = int(mc["realizations"])
    cells = [(k, s, m) for k in mc["kappas"] for s in mc["snrs"] for m in mc["methods"]]
    items = [(cells[c][0], cells[c][1], c * r + i) for c in range(len(cells)) for i in range(r)]
    drawn = S._draw_all(base, grid, setup, items, workers=1)
    assert np.array_equal(np.stack([d[0] for d in drawn]), mc[f"{tag}/pixels"])
    assert np.array_equal(np.array([d[1] for d in drawn], dtype=np.uint64), mc[f"{tag}/seeds"])


def test_wilson_matches_reference_cells(mc):
    r = int(mc["realizations"])
    for tag in ("phi0", "phirand"):
        hits = mc[f"{tag}/outcomes"].sum(axis=1)
        ci = np.array([S.wilson_interval(int(h), r) for h in hits])
        assert np.array_equal(ci, mc[f"{tag}/ci"])
        assert np.array_equal(hits / r, mc[f"{tag}/p_d"])


def test_wilson_edges():
    lo, hi = S.wilson_interval(0, 10)
    assert lo == 0.0 and 0 < hi < 1
    lo, hi = S.wilson_interval(10, 10)
    assert hi == pytest.approx(1.0) and 0 < lo < 1
    with pytest.raises(ConfigurationError):
        S.wilson_interval(0, 0)


def test_detection_criterion():
    geom = S.demo_geometry()
    truth = S.Scenario(geometry=geom, scatterers=(S.Scatterer(-1.0), S.Scatterer(2.0)), snr_db=(10.0, 10.0))

    class Est:
        def __init__(self, k, e):
            self.model_order, self.elevations = k, np.array(e)

    assert S.detection_criterion(Est(2, [2.1, -0.9]), truth, tol=0.2)
    assert not S.detection_criterion(Est(2, [2.1, -0.5]), truth, tol=0.2)
    assert not S.detection_criterion(Est(1, [2.0]), truth, tol=0.2)
    with pytest.raises(ConfigurationError):
        S.detection_criterion(Est(2, [0, 0]), truth, tol=0.0)


def test_synthesize_noise_free_is_steering_sum():
    geom = S.demo_geometry()
    sc = (S.Scatterer(1.5, amplitude=2.0, phase=0.3),)
    truth = S.Scenario(geometry=geom, scatterers=sc, snr_db=(np.inf,))
    g = S.synthesize_pixel(truth, S.substream(0, 0))
    assert np.allclose(g, 2.0 * np.exp(0.3j) * steering_column(geom, 1.5))


def test_validation():
    geom = S.demo_geometry()
    with pytest.raises(ConfigurationError):
        S.Scenario(geometry=geom, scatterers=(S.Scatterer(0.0),), snr_db=())
    with pytest.raises(ConfigurationError):
        S.Scatterer(0.0, amplitude=-1.0)
    with pytest.raises(ConfigurationError):
        S.MonteCarloSetup(grid_size=2)
    with pytest.raises(GeometryError):
        AcquisitionGeometry(np.array([0.0, 0.0]), np.array([0.0, 1.0]), 0.031, 6e5)
    with pytest.raises(ConfigurationError):
        S.monte_carlo_detection(S.Scenario(geometry=geom), [1.0], [10.0], ["fista"], 0)


def test_results_csv(tmp_path):
    res = [S.DetectionResult(0.5, 6.0, "fista", 0.25, 4, 0.04, 0.7)]
    p = tmp_path / "r.csv"
    S.results_to_csv(res, p)
    assert p.read_text() == "kappa,snr_db,method,p_d,ci_low,ci_high,n\n0.5,6.0,fista,0.25,0.04,0.7,4\n"
