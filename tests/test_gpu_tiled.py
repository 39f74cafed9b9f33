"""GPU parity of the large-dictionary (tiled) solver and of the column-sharded multi-GPU algorithm
(emulated with several shards on one device), against the reference golden vectors and the
fp64 oracle.  Tolerances as in test_gpu_parity.py."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import batch as OB  # noqa: E402
from oracle import tomo_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def tb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1805_01759_b200 as tb

    return tb


@pytest.mark.parametrize("backend", ["rbpg", "fista", "ista"])
def test_tiled_matches_golden_cfg1(tb, golden, backend):
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


def _motion_problem(tb, seed=5, ns=40, nv=10, nd=10, p=16):
    from paper_1805_01759_b200.synth import motion_dictionary

    rng = np.random.default_rng(seed)
    freqs = np.sort(rng.uniform(-0.5, 0.5, 100))
    times = np.sort(rng.uniform(0, 4, 100))
    grid = tb.ParameterGrid(elevation=(np.arange(ns) - ns // 2) * 0.25, motion_axes=(np.linspace(-0.02, 0.02, nv), np.linspace(0, 0.01, nd)), motion_bases=("linear", "seasonal"))
    a = motion_dictionary(freqs, times, grid).astype(np.complex64)
    pos = rng.integers(0, a.shape[1], (p, 2))
    a128 = a.astype(np.complex128)
    b = a128[:, pos[:, 0]].T + 0.7 * a128[:, pos[:, 1]].T
    b = (b + 0.3 * (rng.standard_normal(b.shape) + 1j * rng.standard_normal(b.shape))).astype(np.complex64)
    return a, b, grid


@pytest.mark.parametrize("backend", ["rbpg", "fista"])
def test_tiled_motion_grid_vs_oracle(tb, backend):
    a, b, grid = _motion_problem(tb)
    d = tb.Dictionary(a)
    lam = d.default_lambda(b, 0.1).cpu().numpy()
    seeds = d.derive_seeds(3, b.shape[0]).cpu().numpy()
    cfg = tb.SolverConfig(max_iters=80, tol=1e-6, num_blocks=8)
    bs = d.solve(b, lam, cfg, backend, seeds=seeds, path="tiled")
    lips = d.partition(8).lipschitz if backend == "rbpg" else d.lipschitz()
    ref = OB.run(a.astype(np.complex128), b, lam, backend, seeds=seeds, lips=lips, want_x=True, max_iters=80, tol=1e-6, num_blocks=8)
    assert np.array_equal(bs.iterations.cpu().numpy(), [r["iterations"] for r in ref])
    np.testing.assert_allclose(bs.objective_final.cpu().numpy(), [r["f_final"] for r in ref], rtol=1e-6)
    rx = np.array([r["x_hat"] for r in ref])
    err = np.linalg.norm(bs.x_hat.cpu().numpy() - rx, axis=1) / np.linalg.norm(rx, axis=1)
    assert err.max() <= 1e-4
    # the library's automatic path choice (C++ round loop) is the same solver
    bs2 = d.solve(b, lam, cfg, backend, seeds=seeds)
    assert torch.equal(bs2.objective_final, bs.objective_final)
    # selection on the motion grid (joint argmax over motion bins) vs the oracle
    est = tb.select_batch(d, bs.x_hat, b, grid, 2)
    g = OB.GridDesc(grid.elevation, grid.motion_axes)
    for p in range(b.shape[0]):
        ro = O.detect_support(rx[p], g.shape, 2)
        k, sup, _ = O.model_select(a.astype(np.complex128), b[p].astype(np.complex128), ro, 2, 5)
        assert list(est.support[p, : int(est.model_order[p])].cpu().numpy()) == list(sup)


@pytest.mark.parametrize("backend,world", [("rbpg", 2), ("rbpg", 4), ("fista", 2), ("fista", 3)])
def test_column_sharded_emulation(tb, backend, world):
    """The cfg5 multi-GPU algorithm with `world` column shards on one device == unsharded solve."""
    from paper_1805_01759_b200.sharded import ColumnShard, column_shards, gather_columns, local_columns, solve_column_sharded

    a, b, _ = _motion_problem(tb, seed=9, p=12)
    m = a.shape[1]
    full = tb.Dictionary(a)
    lam = full.default_lambda(b, 0.1).cpu().numpy()
    seeds = full.derive_seeds(11, b.shape[0]).cpu().numpy()
    cfg = tb.SolverConfig(max_iters=60, tol=1e-6, num_blocks=8)
    ref = full.solve(b, lam, cfg, backend, seeds=seeds, path="tiled")
    lips = full.partition(8).lipschitz if backend == "rbpg" else full.lipschitz()
    shards_r = column_shards(m, world, 8 if backend == "rbpg" else None)
    shards = [ColumnShard(a[:, local_columns(r)], r, backend, 8, lips) for r in shards_r]
    outs = solve_column_sharded(shards, b, lam, cfg, seeds=seeds)
    for o in outs:
        assert torch.equal(o.iterations, ref.iterations)
        assert torch.equal(o.status, ref.status)
        np.testing.assert_allclose(o.objective_final.cpu().numpy(), ref.objective_final.cpu().numpy(), rtol=1e-10)
    x = gather_columns([o.x_hat.cpu().numpy() for o in outs], shards_r, m)
    np.testing.assert_allclose(x, ref.x_hat.cpu().numpy(), rtol=1e-5, atol=1e-6)


def test_cfg4_subset_vs_oracle(tb):
    from paper_1805_01759_b200.synth import make_config

    c4 = make_config(4, num_pixels=6)
    d = tb.Dictionary(c4.dictionary)
    a = c4.dictionary.astype(np.complex128)
    part = d.partition(8)
    # device power iteration vs the oracle's on one full-size block (solver.py:167-188)
    s, e = part.blocks[3]
    assert part.lipschitz[3] == pytest.approx(2.0 * O.spectral_sq_norm(a[:, s:e]), rel=1e-9)
    lam = d.default_lambda(c4.pixels, 0.1).cpu().numpy()
    seeds = d.derive_seeds(2018, 6).cpu().numpy()
    cfg = tb.SolverConfig(fixed_iters=25, num_blocks=8, tol=1e-6)
    bs = d.solve(c4.pixels, lam, cfg, "rbpg", seeds=seeds)
    ref = OB.run(a, c4.pixels, lam, "rbpg", seeds=seeds, lips=part.lipschitz, want_x=True, fixed_iters=25, tol=1e-6, num_blocks=8, workers=6)
    np.testing.assert_allclose(bs.objective_final.cpu().numpy(), [r["f_final"] for r in ref], rtol=1e-7)
    rx = np.array([r["x_hat"] for r in ref])
    err = np.linalg.norm(bs.x_hat.cpu().numpy() - rx, axis=1) / np.linalg.norm(rx, axis=1)
    assert err.max() <= 1e-4


def test_cfg5_power_iteration_and_rbpg_rhs(tb):
    from paper_1805_01759_b200.synth import make_config

    c5 = make_config(5, num_pixels=2)
    d = tb.Dictionary(c5.dictionary)
    a = c5.dictionary.astype(np.complex128)
    m = a.shape[1]
    # multi-CTA host-driven power iteration on the full 100 x 1,048,576 matrix, 12 fixed steps
    got = d.spectral_sq_norms([(0, m)], max_iter=12, rtol=0.0)[0]
    ref = O.spectral_sq_norm(a, max_iter=12, rtol=0.0)
    assert got == pytest.approx(ref, rel=1e-12)
    part = d.partition(8)
    lam = d.default_lambda(c5.pixels, 0.1).cpu().numpy()
    seeds = d.derive_seeds(2018, 2).cpu().numpy()
    cfg = tb.SolverConfig(fixed_iters=12, num_blocks=8, tol=1e-6)
    bs = d.solve(c5.pixels, lam, cfg, "rbpg", seeds=seeds)
    ref = OB.run(a, c5.pixels, lam, "rbpg", seeds=seeds, lips=part.lipschitz, want_x=True, fixed_iters=12, tol=1e-6, num_blocks=8, workers=2)
    np.testing.assert_allclose(bs.objective_final.cpu().numpy(), [r["f_final"] for r in ref], rtol=1e-7)
    rx = np.array([r["x_hat"] for r in ref])
    err = np.linalg.norm(bs.x_hat.cpu().numpy() - rx, axis=1) / np.linalg.norm(rx, axis=1)
    assert err.max() <= 1e-4


@pytest.mark.parametrize("backend", ["rbpg", "fista", "ista"])
def test_tiled_solver_edges(tb, golden, backend):
    """Closed form, zero measurement, fixed_iters, alpha_init_scale=4 and line-search failure on the
    tiled path, against the reference golden vectors (test_solver.py:185-247)."""

    def solve(a, b, lam, cfg):
        d = tb.Dictionary(np.asarray(a))
        seeds = np.array([int(cfg.seed)], dtype=np.uint64)
        return d.solve(np.asarray(b).reshape(1, -1), np.array([lam]), cfg, backend, seeds=seeds, history=True, path="tiled").solution(0)

    sol = solve(np.eye(6), golden["edge/eye_b"], 0.5, tb.SolverConfig(num_blocks=2, max_iters=2000, tol=1e-12))
    np.testing.assert_allclose(sol.x_hat, golden[f"edge/eye_{backend}_x"], atol=2e-6)
    sol = solve(np.eye(4), np.zeros(4), 0.5, tb.SolverConfig(num_blocks=2, max_iters=50))
    assert tb.solver.STATUS_BY_CODE.index(sol.status) == int(golden[f"edge/zero_{backend}_status"])
    np.testing.assert_array_equal(sol.objective_history, golden[f"edge/zero_{backend}_hist"])
    if backend == "ista":
        return
    a, b, lam = golden["cfg1/a"], golden["cfg1/b"][3], float(golden["cfg1/lam"][3])
    sol = solve(a, b, lam, tb.SolverConfig(num_blocks=8, fixed_iters=37, tol=1e-1, seed=9))
    assert sol.iterations_used == 37
    np.testing.assert_allclose(sol.objective_history, golden[f"edge/fixed_{backend}_hist"], rtol=1e-5)
    sol = solve(a, b, lam, tb.SolverConfig(num_blocks=8, max_iters=60, tol=1e-6, alpha_init_scale=4.0, seed=9))
    ref = golden[f"edge/scale4_{backend}_hist"]
    assert sol.objective_history.size == ref.size
    np.testing.assert_allclose(sol.objective_history, ref, rtol=1e-4)
    sol = solve(a, b, lam, tb.SolverConfig(num_blocks=8, max_iters=60, tol=1e-6, alpha_init_scale=1e30, c_alpha=0.999999, seed=9))
    assert sol.status == tb.SolverStatus.LINE_SEARCH_FAILURE
    assert sol.iterations_used == int(golden[f"edge/lsfail_{backend}_iters"])
    np.testing.assert_allclose(sol.objective_history, golden[f"edge/lsfail_{backend}_hist"], rtol=1e-6)


def test_cfg5_selection_kmax3_vs_oracle(tb):
    """k_max = 3 on the 256 x 64 x 64 motion grid: joint argmax decode and BIC with p = 5."""
    from paper_1805_01759_b200.synth import make_config

    c5 = make_config(5, num_pixels=3)
    d = tb.Dictionary(c5.dictionary)
    rng = np.random.default_rng(1)
    m = c5.m
    x = np.zeros((3, m), np.complex64)
    for p in range(3):  # sparse profiles with a few peaks, plus the true support
        idx = rng.choice(m, 12, replace=False)
        x[p, idx] = (rng.standard_normal(12) + 1j * rng.standard_normal(12)).astype(np.complex64)
        x[p, c5.truth_support[p]] = 3.0 + 0.1 * np.arange(len(c5.truth_support[p]))  # no exact ties (numpy argsort order on ties is implementation-defined)
    est = tb.select_batch(d, torch.from_numpy(x).cuda(), c5.pixels, c5.grid, 3)
    a = c5.dictionary.astype(np.complex128)
    for p in range(3):
        cands = O.detect_support(x[p].astype(np.complex128), c5.grid.shape, 3)
        k, sup, sc = O.model_select(a, c5.pixels[p].astype(np.complex128), cands, 3, 5)
        ref = O.estimate_params(a, c5.pixels[p].astype(np.complex128), c5.grid, sup)
        k_gpu = int(est.model_order[p])
        assert k_gpu == k
        assert list(est.support[p, :k].cpu().numpy()) == list(sup)
        np.testing.assert_allclose(est.amplitudes[p, :k].cpu().numpy(), ref["amplitudes"], rtol=1e-9)
        np.testing.assert_allclose(est.elevations[p, :k].cpu().numpy(), ref["elevations"])
        np.testing.assert_allclose(est.motion_params[p, :k].cpu().numpy(), ref["motion_params"])
        np.testing.assert_allclose(est.selection_scores[p, : k + 1].cpu().numpy()[: len(sc)], sc[: k + 1], rtol=1e-10)


def test_device_steering_matrix(tb, golden):
    """On-device dictionary build vs the reference's build_steering_matrix (golden) and vs the host
    synthesis of BASELINE cfg4 (sign -1): equal at complex64 precision."""
    from paper_1805_01759_b200.grid import build_steering_matrix
    from paper_1805_01759_b200.synth import WAVELENGTH, make_config

    g = tb.ParameterGrid(elevation=golden["steer/elev"], motion_axes=(golden["steer/ax0"], golden["steer/ax1"]), motion_bases=("linear", "seasonal"))
    a = build_steering_matrix(golden["steer/xi"], g, eta=golden["steer/eta"], sign=1.0).cpu().numpy()
    ref = golden["steer/a"].astype(np.complex64)
    assert np.max(np.abs(a - ref)) <= 2.5e-7
    c4 = make_config(4, num_pixels=1)
    f, t = c4.meta["freqs"], c4.meta["times"]
    eta = np.stack([2.0 * t / WAVELENGTH, 2.0 * np.sin(2.0 * np.pi * t) / WAVELENGTH])
    a4 = build_steering_matrix(f, c4.grid, eta=eta, sign=-1.0).cpu().numpy()
    diff = np.abs(a4 - c4.dictionary)
    assert diff.max() <= 2.5e-7
    assert np.mean(a4 == c4.dictionary) > 0.999
    # a column shard is the same columns of the full build
    shard = build_steering_matrix(f, c4.grid, eta=eta, sign=-1.0, col_range=(1000, 5000)).cpu().numpy()
    np.testing.assert_array_equal(shard, a4[:, 1000:5000])
