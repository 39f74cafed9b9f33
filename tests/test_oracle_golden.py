"""Pin the CPU oracle against fixtures produced by the real reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from oracle import tomo_oracle as O

STATUS = {v: k for k, v in O.STATUS_CODES.items()}


def test_soft_threshold(golden):
    v, taus, out = golden["soft/v"], golden["soft/tau"], golden["soft/out"]
    for t, o in zip(taus, out):
        np.testing.assert_allclose(O.soft_threshold(v, float(t)), o, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("case", range(4))
def test_prox_machinery(golden, case):
    g = lambda k: golden[f"prox{case}/{k}"]  # noqa: E731
    a, b, lam, x = g("a"), g("b"), float(g("lam")), g("x")
    assert O.eval_f(a, b, x) == pytest.approx(float(g("f")), rel=1e-13)
    assert O.eval_F(a, b, lam, x) == pytest.approx(float(g("F")), rel=1e-13)
    np.testing.assert_allclose(O.grad_f(a, b, x), g("grad"), rtol=1e-12)
    lip = 2.0 * O.spectral_sq_norm(a)
    assert lip == pytest.approx(float(g("lip")), rel=1e-13)
    np.testing.assert_allclose(O.prox_step(a, b, lam, x, 0.7 / lip), g("prox"), rtol=1e-12, atol=1e-14)
    assert O.line_search_ok(a, b, x, O.prox_step(a, b, lam, x, 1.0 / lip), 1.0 / lip) == bool(g("ls_safe"))
    assert O.line_search_ok(a, b, x, O.prox_step(a, b, lam, x, 50.0 / lip), 50.0 / lip) == bool(g("ls_big"))
    al, xn = O.backtrack(a, b, lam, x, 16.0 / lip, 0.5)
    assert al == float(g("bt_alpha"))
    np.testing.assert_allclose(xn, g("bt_x"), rtol=1e-12, atol=1e-14)
    assert O.default_lambda(a, b) == pytest.approx(float(g("deflam")), rel=1e-14)
    assert O.default_lambda(a, b, 0.3) == pytest.approx(float(g("deflam3")), rel=1e-14)


@pytest.mark.parametrize("case", range(4))
def test_spectral_norm(golden, case):
    assert O.spectral_sq_norm(golden[f"spec{case}/a"]) == pytest.approx(float(golden[f"spec{case}/s2"]), rel=1e-13)


@pytest.mark.parametrize("j", [1, 3, 8])
def test_partition(golden, j):
    a = golden["cfg1/a"].astype(np.complex128)
    ranges = O.block_ranges(a.shape[1], j)
    assert np.array_equal(np.array(ranges), golden[f"part{j}/blocks"])
    lip = O.block_lipschitz(a, ranges)
    np.testing.assert_allclose(lip, golden[f"part{j}/lip"], rtol=1e-13)
    np.testing.assert_allclose(O.block_probabilities(lip), golden[f"part{j}/prob"], rtol=1e-13)


def test_philox_and_draws(golden):
    assert [int(v) for v in golden["philox/raw"]] == O.philox_raw(987654321, 42, 12)
    cdf = O.choice_cdf(golden["part8/prob"])
    for seed in (0, 7, 123456789, 2**62 + 11):
        s = O.BlockSampler(cdf, seed)
        assert [s.draw() for _ in range(256)] == list(golden[f"draws/{seed}"])


def test_derive_seed(golden):
    for s, row in zip(golden["seeds/run"], golden["seeds/derived"]):
        assert [O.derive_seed(int(s), pid) for pid in range(64)] == [int(v) for v in row]


@pytest.mark.parametrize("backend", ["rbpg", "fista", "ista"])
def test_cfg1_solvers_and_pipeline(golden, backend):
    a = golden["cfg1/a"].astype(np.complex128)
    pix, lam, seeds = golden["cfg1/b"], golden["cfg1/lam"], golden["cfg1/pixel_seeds"]

    class G:
        elevation = golden["cfg1/elev"]
        motion_axes = ()
        shape = (a.shape[1],)

    npx = 8 if backend == "ista" else pix.shape[0]
    for p in range(npx):
        cfg = O.SolverCfg(max_iters=500, tol=1e-6, num_blocks=8, seed=int(seeds[p]))
        est = O.pipeline(a, pix[p].astype(np.complex128), float(lam[p]), G, 2, backend, cfg)
        sol = est["solution"]
        it = int(golden[f"cfg1/{backend}/iters"][p])
        assert sol["iterations"] == it
        assert O.STATUS_CODES[sol["status"]] == int(golden[f"cfg1/{backend}/status"][p])
        np.testing.assert_allclose(sol["history"], golden[f"cfg1/{backend}/hist"][p][: it + 1], rtol=1e-10)
        np.testing.assert_allclose(sol["x_hat"], golden[f"cfg1/{backend}/x"][p], rtol=1e-7, atol=1e-9)
        assert est["model_order"] == int(golden[f"cfg1/{backend}/order"][p])
        sup = golden[f"cfg1/{backend}/support"][p]
        assert list(est["support"]) == [int(v) for v in sup if v >= 0]
        np.testing.assert_allclose(est["amplitudes"], golden[f"cfg1/{backend}/amps"][p][: est["model_order"]], rtol=1e-9)


@pytest.mark.parametrize("backend", ["rbpg", "fista", "ista"])
def test_solver_edges(golden, backend):
    solve = O.SOLVERS[backend]
    sol = solve(np.eye(6), golden["edge/eye_b"], 0.5, O.SolverCfg(num_blocks=2, max_iters=2000, tol=1e-12))
    np.testing.assert_allclose(sol["x_hat"], golden[f"edge/eye_{backend}_x"], atol=1e-12)
    np.testing.assert_allclose(sol["x_hat"], O.soft_threshold(golden["edge/eye_b"], 0.25), atol=1e-8)
    sol = solve(np.eye(4), np.zeros(4), 0.5, O.SolverCfg(num_blocks=2, max_iters=50))
    assert O.STATUS_CODES[sol["status"]] == int(golden[f"edge/zero_{backend}_status"])
    np.testing.assert_array_equal(sol["history"], golden[f"edge/zero_{backend}_hist"])
    if backend == "ista":
        return
    a = golden["cfg1/a"].astype(np.complex128)
    b = golden["cfg1/b"][3].astype(np.complex128)
    lam = float(golden["cfg1/lam"][3])
    sol = solve(a, b, lam, O.SolverCfg(num_blocks=8, fixed_iters=37, tol=1e-1, seed=9))
    assert sol["iterations"] == int(golden[f"edge/fixed_{backend}_iters"]) == 37
    np.testing.assert_allclose(sol["history"], golden[f"edge/fixed_{backend}_hist"], rtol=1e-11)
    sol = solve(a, b, lam, O.SolverCfg(num_blocks=8, max_iters=60, tol=1e-6, alpha_init_scale=4.0, seed=9))
    np.testing.assert_allclose(sol["history"], golden[f"edge/scale4_{backend}_hist"], rtol=1e-10)
    sol = solve(a, b, lam, O.SolverCfg(num_blocks=8, max_iters=60, tol=1e-6, alpha_init_scale=1e30, c_alpha=0.999999, seed=9))
    assert O.STATUS_CODES[sol["status"]] == int(golden[f"edge/lsfail_{backend}_status"]) == 2
    assert sol["iterations"] == int(golden[f"edge/lsfail_{backend}_iters"])
    np.testing.assert_array_equal(sol["history"], golden[f"edge/lsfail_{backend}_hist"])


def test_detect_support(golden):
    for i in range(int(golden["detect/count"])):
        shape = tuple(int(v) for v in golden[f"detect{i}/shape"])
        out = O.detect_support(golden[f"detect{i}/x"], shape, int(golden[f"detect{i}/k"]))
        assert list(out) == list(golden[f"detect{i}/out"]), i


def test_model_select_rank_deficient(golden):
    a = np.array([[1.0, 1.0, 0.0], [0.0, 0.0, 1.0]], dtype=complex)
    k, sup, sc = O.model_select(a, np.array([1.0, 0.5], dtype=complex), np.array([0, 1, 2]), 3)
    assert k == int(golden["msel_dup/k"])
    assert list(sup) == list(golden["msel_dup/support"])
    np.testing.assert_allclose(sc, golden["msel_dup/scores"], rtol=1e-12)


def test_steering_restatement_matches_reference(golden):
    """exp(j 2 pi (xi s + eta_0 p_0 + eta_1 p_1)) row-major over the grid (model.py:296-323)."""
    xi, eta = golden["steer/xi"], golden["steer/eta"]
    s, p0, p1 = golden["steer/elev"], golden["steer/ax0"], golden["steer/ax1"]
    mesh = np.meshgrid(s, p0, p1, indexing="ij")
    phase = np.outer(xi, mesh[0].reshape(-1))
    phase += np.outer(eta[0], mesh[1].reshape(-1))
    phase += np.outer(eta[1], mesh[2].reshape(-1))
    np.testing.assert_array_equal(np.exp(2j * np.pi * phase), golden["steer/a"])


@pytest.mark.parametrize("mu", [0.0, 2.5])
def test_svd_wiener(golden, mu):
    a = golden["cfg1/a"].astype(np.complex128)
    pix = golden["cfg1/b"]

    class G:
        elevation = golden["cfg1/elev"]
        motion_axes = ()
        shape = (a.shape[1],)

    for p in range(pix.shape[0]):
        np.testing.assert_allclose(O.svd_wiener(a, pix[p], mu), golden[f"wiener{mu}/x"][p], rtol=1e-9, atol=1e-12)
        est = O.pipeline(a, pix[p].astype(np.complex128), mu, G, 2, "svd_wiener", None)
        assert list(est["support"]) == [int(v) for v in golden[f"wiener{mu}/support"][p] if v >= 0]
