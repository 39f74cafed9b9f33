"""GPU parity of the tiled solver with the adjoint on the tensor cores (k_tc_tiled.cu,
TB_TILED_TC=1): same golden vectors / oracle bars as test_gpu_tiled.py, plus agreement with the
SIMT-adjoint tiled path on a motion grid whose blocks are not multiples of the 128-column tile."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import batch as OB  # noqa: E402


@pytest.fixture(scope="module")
def tb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1805_01759_b200 as tb

    return tb


@pytest.fixture
def tc_on(monkeypatch):
    monkeypatch.setenv("TB_TILED_TC", "1")


@pytest.mark.parametrize("backend", ["rbpg", "fista", "ista"])
def test_tc_tiled_matches_golden_cfg1(tb, golden, tc_on, backend):
    d = tb.Dictionary(golden["cfg1/a"])
    pix, lam, seeds = golden["cfg1/b"], golden["cfg1/lam"], golden["cfg1/pixel_seeds"]
    bs = d.solve(pix, lam, tb.SolverConfig(max_iters=500, tol=1e-6), backend, seeds=seeds, history=True, path="tiled")
    rit = golden[f"cfg1/{backend}/iters"]
    assert np.array_equal(bs.iterations.cpu().numpy(), rit)
    assert np.array_equal(bs.status.cpu().numpy(), golden[f"cfg1/{backend}/status"])
    rf = np.array([golden[f"cfg1/{backend}/hist"][p][rit[p]] for p in range(len(rit))])
    np.testing.assert_allclose(bs.objective_final.cpu().numpy(), rf, rtol=1e-6)
    rx = golden[f"cfg1/{backend}/x"]
    err = np.linalg.norm(bs.x_hat.cpu().numpy() - rx, axis=1) / np.maximum(np.linalg.norm(rx, axis=1), 1e-30)
    assert err.max() <= 1e-4


def _problem(seed, n, m, p):
    rng = np.random.default_rng(seed)
    a = (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))) / np.sqrt(2 * n)
    pos = rng.integers(0, m, (p, 3))
    b = a[:, pos[:, 0]].T + 0.6 * a[:, pos[:, 1]].T - 0.4j * a[:, pos[:, 2]].T
    b = b + 0.05 * (rng.standard_normal(b.shape) + 1j * rng.standard_normal(b.shape))
    return a.astype(np.complex64), b.astype(np.complex64)


@pytest.mark.parametrize("backend,n,m,p", [("rbpg", 100, 2000, 40), ("fista", 100, 2000, 40), ("rbpg", 37, 1000, 33), ("fista", 70, 777, 65)])
def test_tc_tiled_vs_oracle(tb, tc_on, backend, n, m, p):
    a, b = _problem(n + m + p, n, m, p)
    d = tb.Dictionary(a)
    lam = d.default_lambda(b, 0.1).cpu().numpy()
    seeds = d.derive_seeds(7, p).cpu().numpy()
    cfg = tb.SolverConfig(max_iters=60, tol=1e-6, num_blocks=8)
    bs = d.solve(b, lam, cfg, backend, seeds=seeds, path="tiled")
    lips = d.partition(8).lipschitz if backend == "rbpg" else d.lipschitz()
    ref = OB.run(a.astype(np.complex128), b, lam, backend, seeds=seeds, lips=lips, want_x=True, max_iters=60, tol=1e-6, num_blocks=8)
    assert np.array_equal(bs.iterations.cpu().numpy(), [r["iterations"] for r in ref])
    np.testing.assert_allclose(bs.objective_final.cpu().numpy(), [r["f_final"] for r in ref], rtol=1e-6)
    rx = np.array([r["x_hat"] for r in ref])
    err = np.linalg.norm(bs.x_hat.cpu().numpy() - rx, axis=1) / np.linalg.norm(rx, axis=1)
    assert err.max() <= 1e-4
