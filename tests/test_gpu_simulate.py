"""Batched Monte-Carlo harness on the GPU vs the reference harness's per-realization outcomes
(tests/golden/mc_small.npz).  Pixels are bit-identical (test_simulate.py); the solve runs in
float32 against the reference's float64, so a realization sitting on a detection boundary may
flip.  Bar: >= 95 % of realizations agree per method, and every cell's p_d lies inside the
reference cell's 95 % Wilson interval widened by 2 realizations."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def mc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return np.load(os.path.join(HERE, "golden", "mc_small.npz"))


@pytest.mark.parametrize("tag,dphi", [("phi0", 0.0), ("phirand", None)])
def test_mc_outcomes_vs_reference(mc, tag, dphi):
    from paper_1805_01759_b200 import simulate as S
    from paper_1805_01759_b200.solver import SolverConfig

    r = int(mc["realizations"])
    base = S.Scenario(geometry=S.demo_geometry(), seed=int(mc["seed"]))
    setup = S.MonteCarloSetup(delta_phi=dphi, solver=SolverConfig(max_iters=300, tol=1e-6))
    methods = [str(m) for m in mc["methods"]]
    cells, got = S.monte_carlo_outcomes(base, list(mc["kappas"]), list(mc["snrs"]), methods, r, setup)
    ref = mc[f"{tag}/outcomes"]
    assert got.shape == ref.shape
    agree = got == ref
    for meth in methods:
        rows = [i for i, c in enumerate(cells) if c[2] == meth]
        frac = agree[rows].mean()
        print(tag, meth, "agreement", frac)
        assert frac >= 0.95, (meth, frac)
    res = S.monte_carlo_detection(base, list(mc["kappas"]), list(mc["snrs"]), methods, r, setup)
    for x, (lo, hi) in zip(res, mc[f"{tag}/ci"]):
        assert lo - 2.0 / r <= x.p_d <= hi + 2.0 / r


def test_device_draws_statistics():
    """tb_synthesize_pairs: the noise is circular complex Gaussian with variance sigma^2, a drawn phase
    is uniform on [0, 2 pi), nested seeds are 63-bit and distinct, and draws are deterministic."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1805_01759_b200 import simulate as S
    from paper_1805_01759_b200.geometry import steering_dictionary
    from paper_1805_01759_b200.solver import Dictionary

    base = S.Scenario(geometry=S.demo_geometry(), seed=3)
    setup = S.MonteCarloSetup()
    grid = S.harness_grid(base, setup)
    d = Dictionary(steering_dictionary(base.geometry, grid))
    a = d.tensor.cpu().numpy().astype(np.complex128)
    r = 20000
    ids = np.arange(r, dtype=np.uint64) + 1000
    sigma = 0.7
    pix, seeds = d.synthesize_pairs(base.seed, ids, np.full(r, 40), np.full(r, 90), np.zeros(r, np.float32), np.full(r, sigma, np.float32))
    noise = pix.cpu().numpy().astype(np.complex128) - (a[:, 40] + a[:, 90])[None, :]
    assert abs(noise.real.var() - sigma**2 / 2) <= 0.03 * sigma**2 / 2 and abs(noise.imag.var() - sigma**2 / 2) <= 0.03 * sigma**2 / 2
    assert abs(noise.mean()) <= 0.01 and abs(np.mean(noise.real * noise.imag)) <= 0.01 * sigma**2
    s = seeds.cpu().numpy()
    assert len(np.unique(s)) == r and int(s.max()) < 2**63
    pix2, seeds2 = d.synthesize_pairs(base.seed, ids, np.full(r, 40), np.full(r, 90), np.zeros(r, np.float32), np.full(r, sigma, np.float32))
    assert torch.equal(pix, pix2) and torch.equal(seeds, seeds2)
    # drawn phase, no noise: g = A0 + e^{j phi} A1 -> phi uniform on [0, 2 pi)
    pix3, _ = d.synthesize_pairs(base.seed, ids, np.full(r, 40), np.full(r, 90), np.full(r, np.nan, np.float32), np.zeros(r, np.float32))
    g = pix3.cpu().numpy().astype(np.complex128) - a[:, 40][None, :]
    phi = np.angle(np.sum(g * np.conj(a[:, 90])[None, :], axis=1) / np.vdot(a[:, 90], a[:, 90]).real) % (2 * np.pi)
    hist, _ = np.histogram(phi, bins=8, range=(0, 2 * np.pi))
    assert np.all(np.abs(hist - r / 8) <= 5 * np.sqrt(r / 8))


@pytest.mark.parametrize("dphi", [0.0, None])
def test_device_draws_detection_rates_match_host(dphi):
    """The whole sweep with draws on the device gives the same detection rates as with the
    reference's own host draws (bit-identical to the reference's pixels): every cell within 4 sigma
    of the binomial difference at 1,500 realizations per cell."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1805_01759_b200 import simulate as S
    from paper_1805_01759_b200.solver import SolverConfig

    r = 1500
    base = S.Scenario(geometry=S.demo_geometry(), seed=11)
    setup = S.MonteCarloSetup(delta_phi=dphi, solver=SolverConfig(max_iters=300, tol=1e-6))
    kappas, snrs, methods = [0.6, 1.2], [5.0, 15.0], ["rbpg", "fista", "svd_wiener"]
    host = S.monte_carlo_detection(base, kappas, snrs, methods, r, setup, workers=os.cpu_count() or 1)
    dev = S.monte_carlo_detection(base, kappas, snrs, methods, r, setup, draws="device")
    for h, g in zip(host, dev):
        assert (h.kappa, h.snr_db, h.method) == (g.kappa, g.snr_db, g.method)
        p = (h.p_d + g.p_d) / 2
        assert abs(h.p_d - g.p_d) <= 4 * np.sqrt(max(p * (1 - p), 1.0 / r) * 2 / r) + 1.0 / r, (h, g)
