"""GPU parity: the sm_100a path (through the C ABI) against the reference golden vectors and the
fp64 oracle on the same complex64-rounded inputs.

Tolerances (north_star: support bit-exact; amplitudes/objective within a stated relative
tolerance in complex64):
  * integer/index outputs (seeds, block draws via iteration counts, support, model order): exact
  * objective (final F): relative 1e-4
  * debiased amplitudes: relative 1e-6 (same support -> same fp64 LS)
  * x_hat: relative L2 error median <= 1e-4; FISTA max <= 5e-2 (window-stop jitter of the
    non-monotone method moves the stop iteration), RBPG/ISTA max <= 1e-3
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import batch as OB  # noqa: E402
from oracle import tomo_oracle as O  # noqa: E402

STATUS = {v: k for k, v in O.STATUS_CODES.items()}


@pytest.fixture(scope="module")
def tb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1805_01759_b200 as tb

    return tb


@pytest.fixture(scope="module")
def cfg1(tb, golden):
    d = tb.Dictionary(golden["cfg1/a"])
    return d


def test_seeds_match_reference(tb, golden, cfg1):
    for s, row in zip(golden["seeds/run"], golden["seeds/derived"]):
        got = cfg1.derive_seeds(int(s), 64).cpu().numpy()
        assert np.array_equal(got, row.astype(np.uint64))
    got = cfg1.derive_seeds(2018, 24).cpu().numpy()
    assert np.array_equal(got, golden["cfg1/pixel_seeds"])


def test_lambda_rule(tb, golden, cfg1):
    pix = golden["cfg1/b"]
    lam = cfg1.default_lambda(pix, 0.1).cpu().numpy()
    np.testing.assert_allclose(lam, golden["cfg1/lam"], rtol=1e-5)
    a = golden["cfg1/a"].astype(np.complex128)
    for p in range(4):
        ref = O.default_lambda(a, pix[p].astype(np.complex128), 0.05)
        assert float(cfg1.default_lambda(pix[p : p + 1], 0.05)[0]) == pytest.approx(ref, rel=1e-5)


def test_spectral_norms(tb, golden, cfg1):
    assert cfg1.lipschitz() == pytest.approx(float(golden["cfg1/lip_full"]), rel=1e-10)
    for j in (1, 3, 8):
        part = cfg1.partition(j)
        assert np.array_equal(np.array(part.blocks), golden[f"part{j}/blocks"])
        np.testing.assert_allclose(part.lipschitz, golden[f"part{j}/lip"], rtol=1e-10)
        np.testing.assert_allclose(part.probabilities, golden[f"part{j}/prob"], rtol=1e-10)
    for case in range(4):
        a = golden[f"spec{case}/a"]
        got = tb.spectral_sq_norm(a.astype(np.complex64))
        ref = O.spectral_sq_norm(a.astype(np.complex64).astype(np.complex128))
        assert got == pytest.approx(ref, rel=1e-9)


@pytest.mark.parametrize("backend", ["rbpg", "fista", "ista"])
def test_golden_cfg1_solvers(tb, golden, cfg1, backend):
    pix, lam, seeds = golden["cfg1/b"], golden["cfg1/lam"], golden["cfg1/pixel_seeds"]
    cfg = tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8)
    bs = cfg1.solve(pix, lam, cfg, backend, seeds=seeds, history=True)
    it = bs.iterations.cpu().numpy()
    st = bs.status.cpu().numpy()
    x = bs.x_hat.cpu().numpy()
    ff = bs.objective_final.cpu().numpy()
    rit, rst, rx = golden[f"cfg1/{backend}/iters"], golden[f"cfg1/{backend}/status"], golden[f"cfg1/{backend}/x"]
    rf = np.array([golden[f"cfg1/{backend}/hist"][p][rit[p]] for p in range(len(rit))])
    # every solver (FISTA included: its extrapolation memory is fp64, so y and A y agree) stops at
    # the reference's iteration with the reference's status on every golden pixel
    assert np.array_equal(st, rst)
    assert np.array_equal(it, rit)
    np.testing.assert_allclose(ff, rf, rtol=1e-4)
    err = np.linalg.norm(x - rx, axis=1) / np.maximum(np.linalg.norm(rx, axis=1), 1e-30)
    assert np.median(err) <= 1e-4
    assert err.max() <= 1e-3
    # early history (before trajectories can drift) tracks the reference closely
    h = bs.history.cpu().numpy()
    k = 30
    np.testing.assert_allclose(h[:, :k], golden[f"cfg1/{backend}/hist"][:, :k], rtol=1e-5)
    grid = tb.ParameterGrid(elevation=golden["cfg1/elev"])
    est = tb.select_batch(cfg1, bs.x_hat, pix, grid, 2)
    assert np.array_equal(est.model_order.cpu().numpy(), golden[f"cfg1/{backend}/order"])
    assert np.array_equal(est.support.cpu().numpy(), golden[f"cfg1/{backend}/support"])
    np.testing.assert_allclose(est.amplitudes.cpu().numpy(), golden[f"cfg1/{backend}/amps"], rtol=1e-6, atol=1e-12)
    sc, rsc = est.selection_scores.cpu().numpy(), golden[f"cfg1/{backend}/scores"]
    assert np.array_equal(np.isnan(sc), np.isnan(rsc))
    np.testing.assert_allclose(sc[~np.isnan(sc)], rsc[~np.isnan(rsc)], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("backend", ["rbpg", "fista"])
def test_solver_edges(tb, golden, backend):
    eye = tb.Objective(dictionary=np.eye(6), measurement=golden["edge/eye_b"], lambda_reg=0.5)
    sol = {"rbpg": tb.rbpg_solve, "fista": tb.fista_solve}[backend](eye, tb.SolverConfig(num_blocks=2, max_iters=2000, tol=1e-12))
    np.testing.assert_allclose(sol.x_hat, golden[f"edge/eye_{backend}_x"], atol=2e-6)
    zero = tb.Objective(dictionary=np.eye(4), measurement=np.zeros(4), lambda_reg=0.5)
    sol = {"rbpg": tb.rbpg_solve, "fista": tb.fista_solve}[backend](zero, tb.SolverConfig(num_blocks=2, max_iters=50))
    assert sol.status.value == STATUS[int(golden[f"edge/zero_{backend}_status"])]
    np.testing.assert_array_equal(sol.objective_history, golden[f"edge/zero_{backend}_hist"])
    a = golden["cfg1/a"]
    obj = tb.Objective(dictionary=a.astype(np.complex128), measurement=golden["cfg1/b"][3], lambda_reg=float(golden["cfg1/lam"][3]))
    solve = {"rbpg": tb.rbpg_solve, "fista": tb.fista_solve}[backend]
    sol = solve(obj, tb.SolverConfig(num_blocks=8, fixed_iters=37, tol=1e-1, seed=9))
    assert sol.iterations_used == 37
    assert sol.status.value == STATUS[int(golden[f"edge/fixed_{backend}_status"])]
    np.testing.assert_allclose(sol.objective_history, golden[f"edge/fixed_{backend}_hist"], rtol=1e-5)
    sol = solve(obj, tb.SolverConfig(num_blocks=8, max_iters=60, tol=1e-6, alpha_init_scale=4.0, seed=9))
    ref = golden[f"edge/scale4_{backend}_hist"]
    assert sol.objective_history.size == ref.size
    np.testing.assert_allclose(sol.objective_history, ref, rtol=1e-4)
    sol = solve(obj, tb.SolverConfig(num_blocks=8, max_iters=60, tol=1e-6, alpha_init_scale=1e30, c_alpha=0.999999, seed=9))
    assert sol.status == tb.SolverStatus.LINE_SEARCH_FAILURE
    assert sol.iterations_used == int(golden[f"edge/lsfail_{backend}_iters"])
    np.testing.assert_allclose(sol.objective_history, golden[f"edge/lsfail_{backend}_hist"], rtol=1e-6)


def _cfg_batch(tb, cfg_id, npx):
    from paper_1805_01759_b200.synth import make_config

    return make_config(cfg_id, num_pixels=npx)


@pytest.mark.parametrize("cfg_id,npx,backends", [(1, 1024, ("rbpg", "fista")), (2, 256, ("rbpg", "fista")), (3, 96, ("rbpg", "fista"))])
def test_pipeline_vs_oracle(tb, cfg_id, npx, backends):
    """Full pipeline at the BASELINE settings on the GPU vs the oracle on the same inputs."""
    batch = _cfg_batch(tb, cfg_id, npx)
    d = tb.Dictionary(batch.dictionary)
    a = batch.dictionary.astype(np.complex128)
    grid = OB.GridDesc(batch.grid.elevation, batch.grid.motion_axes)
    for backend in backends:
        pc = tb.PipelineConfig(solver=tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018), backend=backend, k_max=batch.k_max)
        est = tb.pipeline_batch(d, batch.pixels, batch.grid, pc, beta=0.1)
        lam = est.lam.cpu().numpy()
        seeds = d.derive_seeds(2018, npx).cpu().numpy()
        lips = d.partition(8).lipschitz if backend == "rbpg" else d.lipschitz()
        ref = OB.run(a, batch.pixels, lam, backend, seeds=seeds, grid=grid, k_max=batch.k_max, lips=lips, max_iters=500, tol=1e-6, num_blocks=8)
        sup = est.support.cpu().numpy()
        order = est.model_order.cpu().numpy()
        amps = est.amplitudes.cpu().numpy()
        ff = est.solution.objective_final.cpu().numpy()
        mism = [p for p in range(npx) if list(sup[p, : order[p]]) != list(ref[p]["support"])]
        assert not mism, f"{backend} cfg{cfg_id}: support differs on {len(mism)}/{npx} pixels: {mism[:8]}"
        for p in range(npx):
            k = order[p]
            np.testing.assert_allclose(amps[p, :k], ref[p]["amplitudes"], rtol=1e-6, atol=1e-12)
        rf = np.array([r["f_final"] for r in ref])
        np.testing.assert_allclose(ff, rf, rtol=1e-4)


def test_determinism_and_order_independence(tb, cfg1):
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(1, num_pixels=512)
    d = tb.Dictionary(batch.dictionary)
    lam = d.default_lambda(batch.pixels, 0.1)
    seeds = d.derive_seeds(7, 512).view(torch.int64)
    cfg = tb.SolverConfig(max_iters=500, tol=1e-6)
    for backend in ("rbpg", "fista"):
        r1 = d.solve(batch.pixels, lam, cfg, backend, seeds=seeds)
        r2 = d.solve(batch.pixels, lam, cfg, backend, seeds=seeds)
        assert torch.equal(r1.x_hat, r2.x_hat) and torch.equal(r1.objective_final, r2.objective_final)
        perm = torch.randperm(512, generator=torch.Generator().manual_seed(0)).to(lam.device)
        px = torch.from_numpy(batch.pixels).to(lam.device)[perm]
        r3 = d.solve(px, lam[perm], cfg, backend, seeds=seeds[perm])
        assert torch.equal(r3.x_hat, r1.x_hat[perm])
        assert torch.equal(r3.iterations, r1.iterations[perm])
        # split batch (as on 2 GPUs) gives identical per-pixel results
        r4 = d.solve(px[:200], lam[perm][:200], cfg, backend, seeds=seeds[perm][:200])
        assert torch.equal(r4.objective_final, r1.objective_final[perm][:200])


def test_single_pixel_api_matches_batch(tb, golden):
    a = golden["cfg1/a"]
    p = 5
    obj = tb.Objective(dictionary=a.astype(np.complex128), measurement=golden["cfg1/b"][p], lambda_reg=float(golden["cfg1/lam"][p]))
    cfg = tb.SolverConfig(max_iters=500, tol=1e-6, seed=int(golden["cfg1/pixel_seeds"][p]))
    sol = tb.rbpg_solve(obj, cfg)
    assert sol.iterations_used == int(golden["cfg1/rbpg/iters"][p])
    assert sol.objective_history.size == sol.iterations_used + 1
    np.testing.assert_allclose(sol.x_hat, golden["cfg1/rbpg/x"][p], rtol=1e-3, atol=1e-5)
    grid = tb.ParameterGrid(elevation=golden["cfg1/elev"])
    est = tb.slimmer_pipeline(obj, grid, tb.PipelineConfig(solver=cfg, backend="rbpg"))
    assert list(est.support) == [int(v) for v in golden["cfg1/rbpg/support"][p] if v >= 0]


def test_empty_and_invalid(tb, cfg1):
    cfg = tb.SolverConfig(max_iters=10)
    r = cfg1.solve(np.zeros((0, cfg1.n), np.complex64), np.zeros(0, np.float32), cfg, "fista")
    assert r.x_hat.shape == (0, cfg1.m)
    with pytest.raises(tb.ConfigurationError):
        cfg1.solve(np.zeros((2, cfg1.n + 1), np.complex64), np.ones(2, np.float32), cfg, "fista")
    with pytest.raises(tb.ConfigurationError):
        cfg1.solve(np.zeros((2, cfg1.n), np.complex64), -np.ones(2, np.float32), cfg, "fista")
    with pytest.raises(tb.ConfigurationError):
        tb.pipeline_batch(cfg1, np.zeros((1, cfg1.n), np.complex64), tb.ParameterGrid(elevation=np.arange(cfg1.m + 1.0)), tb.PipelineConfig(backend="fista"))


def test_large_batch_properties(tb):
    """cfg2-shaped batch at scale: statuses valid, RBPG objective never increases, F <= F0."""
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(2, num_pixels=1 << 16)
    d = tb.Dictionary(batch.dictionary)
    lam = d.default_lambda(batch.pixels, 0.1)
    cfg = tb.SolverConfig(max_iters=500, tol=1e-6)
    r = d.solve(batch.pixels, lam, cfg, "rbpg", seeds=d.derive_seeds(2018, 1 << 16))
    st = r.status.cpu().numpy()
    assert set(np.unique(st)) <= {0, 1}
    b = torch.from_numpy(batch.pixels).to(lam.device)
    f0 = (b.abs() ** 2).sum(dim=1).double()
    assert bool((r.objective_final <= f0 * (1 + 1e-6)).all())
    assert bool(torch.isfinite(r.x_hat).all())


@pytest.mark.parametrize("mu", [0.0, 2.5])
def test_svd_wiener_backend(tb, golden, cfg1, mu):
    """Batched svd_wiener (device SVD filter + apply kernel) and its pipeline vs the reference."""
    pix = golden["cfg1/b"]
    x = cfg1.wiener(pix, mu).cpu().numpy()
    ref = golden[f"wiener{mu}/x"]
    err = np.linalg.norm(x - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= 1e-5
    grid = tb.ParameterGrid(elevation=golden["cfg1/elev"])
    est = tb.pipeline_batch(cfg1, pix, grid, tb.PipelineConfig(backend="svd_wiener", wiener_mu=mu, k_max=2))
    assert np.array_equal(est.support.cpu().numpy(), golden[f"wiener{mu}/support"])
    assert np.array_equal(est.model_order.cpu().numpy(), golden[f"wiener{mu}/order"])
    obj = tb.Objective(dictionary=golden["cfg1/a"].astype(np.complex128), measurement=pix[0], lambda_reg=0.0)
    np.testing.assert_allclose(tb.svd_wiener_solve(obj, mu), ref[0], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("num_blocks", [1, 5, 13, 40])
def test_rbpg_block_counts_vs_oracle(tb, num_blocks):
    """RBPG with block counts other than the default 8 (the per-block delta cache, the block
    table and the column-pass dispatch all depend on J): iterations and statuses identical to the
    oracle, objective within 1e-6."""
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(1, num_pixels=48)
    d = tb.Dictionary(batch.dictionary)
    lam = d.default_lambda(batch.pixels, 0.1)
    seeds = d.derive_seeds(2018, 48)
    cfg = tb.SolverConfig(max_iters=300, tol=1e-6, num_blocks=num_blocks)
    r = d.solve(batch.pixels, lam, cfg, "rbpg", seeds=seeds)
    lips = d.partition(num_blocks).lipschitz
    ref = OB.run(batch.dictionary.astype(np.complex128), batch.pixels, lam.cpu().numpy(), "rbpg", seeds=seeds.cpu().numpy(),
                 lips=lips, max_iters=300, tol=1e-6, num_blocks=num_blocks)
    assert np.array_equal(r.iterations.cpu().numpy(), np.array([x["iterations"] for x in ref]))
    assert np.array_equal(r.status.cpu().numpy(), np.array([O.STATUS_CODES[x["status"]] if isinstance(x["status"], str) else x["status"] for x in ref]))
    np.testing.assert_allclose(r.objective_final.cpu().numpy(), np.array([x["f_final"] for x in ref]), rtol=1e-6)


def test_full_size_cfg2_sampled_vs_oracle(tb):
    """The BASELINE cfg2 batch at full size (1,048,576 pixels, RBPG, the bench's settings): 192
    pixels sampled across the whole batch (including the last ones, whose seeds come from large
    pixel ids) match the oracle exactly in iterations, status and support, objective within 1e-6.
    Nothing is handed from the GPU to the oracle: it computes its own lambda (prox.py:153-161) and,
    as the reference does, its own block partition on every solve (solver.py:267)."""
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(2)
    d = tb.Dictionary(batch.dictionary)
    pc = tb.PipelineConfig(solver=tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018), backend="rbpg", k_max=batch.k_max)
    est = tb.pipeline_batch(d, batch.pixels, batch.grid, pc, beta=0.1)
    rng = np.random.default_rng(7)
    idx = np.sort(np.concatenate([rng.choice(batch.num_pixels, 184, replace=False), np.arange(batch.num_pixels - 8, batch.num_pixels)]))
    idx = np.unique(idx)
    a64 = batch.dictionary.astype(np.complex128)
    lam = np.array([O.default_lambda(a64, batch.pixels[p].astype(np.complex128), 0.1) for p in idx])
    np.testing.assert_allclose(est.lam.cpu().numpy()[idx], lam, rtol=1e-13)
    seeds = np.array([O.derive_seed(2018, int(p)) for p in idx], dtype=np.uint64)
    grid = OB.GridDesc(batch.grid.elevation, batch.grid.motion_axes)
    ref = OB.run(a64, batch.pixels[idx], lam, "rbpg", seeds=seeds, grid=grid, k_max=batch.k_max,
                 lips=None, max_iters=500, tol=1e-6, num_blocks=8)
    its = est.solution.iterations.cpu().numpy()[idx]
    st = est.solution.status.cpu().numpy()[idx]
    ff = est.solution.objective_final.cpu().numpy()[idx]
    sup = est.support.cpu().numpy()[idx]
    order = est.model_order.cpu().numpy()[idx]
    assert np.array_equal(its, np.array([r["iterations"] for r in ref]))
    assert np.array_equal(st, np.array([O.STATUS_CODES[r["status"]] if isinstance(r["status"], str) else r["status"] for r in ref]))
    np.testing.assert_allclose(ff, np.array([r["f_final"] for r in ref]), rtol=1e-6)
    for k in range(len(idx)):
        assert list(sup[k, : order[k]]) == list(ref[k]["support"]), (int(idx[k]), sup[k], ref[k]["support"])


@pytest.mark.parametrize("cfg_id,backend", [(3, "rbpg"), (2, "fista"), (3, "fista")])
def test_full_size_sampled_vs_oracle(tb, cfg_id, backend):
    """Full-size BASELINE batches (cfg2 1,048,576 px / cfg3 262,144 px) solved on the GPU; 96
    pixels sampled across the batch match the oracle in iterations, status and support."""
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(cfg_id)
    d = tb.Dictionary(batch.dictionary)
    pc = tb.PipelineConfig(solver=tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018), backend=backend, k_max=batch.k_max)
    est = tb.pipeline_batch(d, batch.pixels, batch.grid, pc, beta=0.1)
    idx = np.unique(np.random.default_rng(cfg_id).choice(batch.num_pixels, 96, replace=False))
    lam = est.lam.cpu().numpy()[idx]
    seeds = np.array([O.derive_seed(2018, int(p)) for p in idx], dtype=np.uint64)
    grid = OB.GridDesc(batch.grid.elevation, batch.grid.motion_axes)
    lips = d.partition(8).lipschitz if backend == "rbpg" else d.lipschitz()
    ref = OB.run(batch.dictionary.astype(np.complex128), batch.pixels[idx], lam, backend, seeds=seeds, grid=grid, k_max=batch.k_max,
                 lips=lips, max_iters=500, tol=1e-6, num_blocks=8)
    assert np.array_equal(est.solution.iterations.cpu().numpy()[idx], np.array([r["iterations"] for r in ref]))
    np.testing.assert_allclose(est.solution.objective_final.cpu().numpy()[idx], np.array([r["f_final"] for r in ref]), rtol=1e-6)
    sup, order = est.support.cpu().numpy()[idx], est.model_order.cpu().numpy()[idx]
    for k in range(len(idx)):
        assert list(sup[k, : order[k]]) == list(ref[k]["support"]), (int(idx[k]), sup[k], ref[k]["support"])


@pytest.mark.parametrize("backend", ["rbpg", "fista"])
def test_oracle_own_lambda_cfg1(tb, backend):
    """No shared lambda: the GPU computes its own fp64 lambda rule, the oracle its own
    (prox.py:153-161 in fp64 on the same complex64 inputs); solves and selection still agree."""
    batch = _cfg_batch(tb, 1, 128)
    d = tb.Dictionary(batch.dictionary)
    a = batch.dictionary.astype(np.complex128)
    pc = tb.PipelineConfig(solver=tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018), backend=backend, k_max=2)
    est = tb.pipeline_batch(d, batch.pixels, batch.grid, pc, beta=0.1)
    lam_gpu = est.lam.cpu().numpy()
    lam_ref = np.array([O.default_lambda(a, batch.pixels[p].astype(np.complex128), 0.1) for p in range(128)])
    np.testing.assert_allclose(lam_gpu, lam_ref, rtol=1e-13)
    seeds = d.derive_seeds(2018, 128).cpu().numpy()
    lips = d.partition(8).lipschitz if backend == "rbpg" else d.lipschitz()
    grid = OB.GridDesc(batch.grid.elevation)
    ref = OB.run(a, batch.pixels, lam_ref, backend, seeds=seeds, grid=grid, k_max=2, lips=lips, max_iters=500, tol=1e-6, num_blocks=8)
    its = est.solution.iterations.cpu().numpy()
    order, sup = est.model_order.cpu().numpy(), est.support.cpu().numpy()
    assert [int(i) for i in its] == [r["iterations"] for r in ref]
    for p in range(128):
        assert list(sup[p, : order[p]]) == list(ref[p]["support"]), p
        np.testing.assert_allclose(est.amplitudes[p, : order[p]].cpu().numpy(), ref[p]["amplitudes"], rtol=1e-6, atol=1e-12)
