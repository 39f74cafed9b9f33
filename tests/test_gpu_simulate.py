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
