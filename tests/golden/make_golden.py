"""Generate tests/golden/golden_v1.npz by running the REAL reference ``tomobpdn``.

Run in the build container (the reference is importable there, not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

Every fixture stores its own inputs, so the tests never depend on the generators used here.
Cases mirror the reference's own tests (pkg/tests/test_prox.py, test_solver.py,
test_slimmer.py) plus cfg1-shaped pixels (BASELINE.json config 1) run through the three
solvers and the SL1MMER pipeline at the BASELINE settings (max_iters=500, tol=1e-6,
lambda = 0.1 max|A^H b| rounded to float32, A and b rounded to complex64).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

import tomobpdn as T  # noqa: E402
from tomobpdn.rng import derive_seed, substream  # noqa: E402

from paper_1805_01759_b200.synth import lambda_from_beta, make_config  # noqa: E402

STATUS = {"converged": 0, "max-iters": 1, "line-search-failure": 2, "numerical-failure": 3}
OUT = {}


def put(name, value):
    OUT[name] = np.asarray(value)


def rand_c(rng, *shape):
    return rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)


def main():
    rng = np.random.Generator(np.random.Philox(key=[424242, 1]))

    # --- prox.py: soft threshold, prox step, line search, backtrack, default lambda
    v = rand_c(rng, 64) * 3.0
    taus = np.array([0.0, 0.1, 0.7, 1.5, 5.0])
    put("soft/v", v)
    put("soft/tau", taus)
    put("soft/out", np.stack([T.soft_threshold(v, float(t)) for t in taus]))
    for case in range(4):
        a = rand_c(rng, 8, 12)
        b = rand_c(rng, 8)
        lam = [0.3, 0.0, 1.2, 0.05][case]
        x = rand_c(rng, 12)
        obj = T.Objective(dictionary=a, measurement=b, lambda_reg=lam)
        lip = 2.0 * T.spectral_sq_norm(a)
        put(f"prox{case}/a", a)
        put(f"prox{case}/b", b)
        put(f"prox{case}/lam", lam)
        put(f"prox{case}/x", x)
        put(f"prox{case}/f", T.eval_f(obj, x))
        put(f"prox{case}/F", T.eval_F(obj, x))
        put(f"prox{case}/grad", T.grad_f(obj, x))
        put(f"prox{case}/lip", lip)
        put(f"prox{case}/prox", T.prox_step(obj, x, 0.7 / lip))
        put(f"prox{case}/ls_safe", T.line_search_ok(obj, x, T.prox_step(obj, x, 1.0 / lip), 1.0 / lip))
        put(f"prox{case}/ls_big", T.line_search_ok(obj, x, T.prox_step(obj, x, 50.0 / lip), 50.0 / lip))
        al, xn = T.backtrack(obj, x, 16.0 / lip, 0.5)
        put(f"prox{case}/bt_alpha", al)
        put(f"prox{case}/bt_x", xn)
        put(f"prox{case}/deflam", T.default_lambda(a, b))
        put(f"prox{case}/deflam3", T.default_lambda(a, b, beta=0.3))

    # --- solver.py: spectral norm, partition, sampling, seeds
    for case, (n, m) in enumerate([(10, 7), (25, 200), (6, 1), (50, 64)]):
        a = rand_c(rng, n, m)
        put(f"spec{case}/a", a)
        put(f"spec{case}/s2", T.spectral_sq_norm(a))
    cfg1 = make_config(1)
    a64 = cfg1.dictionary
    a = a64.astype(np.complex128)
    put("cfg1/a", a64)
    for j in (1, 3, 8):
        part = T.block_partition(a.shape[1], j, a)
        put(f"part{j}/blocks", np.array(part.blocks))
        put(f"part{j}/lip", part.lipschitz)
        put(f"part{j}/prob", part.probabilities)
    put("cfg1/lip_full", 2.0 * T.spectral_sq_norm(a))
    part8 = T.block_partition(a.shape[1], 8, a)
    for seed in (0, 7, 123456789, 2**62 + 11):
        g = substream(seed)
        put(f"draws/{seed}", np.array([T.sample_block(part8, g) for _ in range(256)]))
    run_seeds = [0, 5, 2018, 2**40 + 3]
    put("seeds/run", np.array(run_seeds, dtype=np.uint64))
    put("seeds/derived", np.array([[derive_seed(substream(s, pid)) for pid in range(64)] for s in run_seeds], dtype=np.uint64))
    bg = np.random.Philox(key=[987654321, 42])
    put("philox/raw", np.array([bg.random_raw() for _ in range(12)], dtype=np.uint64))

    # --- cfg1 pixels through the three solvers + pipeline
    npx = 24
    pix = cfg1.pixels[:npx]
    lam = lambda_from_beta(a64, pix, 0.1)
    put("cfg1/b", pix)
    put("cfg1/lam", lam)
    put("cfg1/elev", cfg1.grid.elevation)
    run_seed = 2018
    pseeds = np.array([derive_seed(substream(run_seed, p)) for p in range(npx)], dtype=np.uint64)
    put("cfg1/pixel_seeds", pseeds)
    grid = T.ParameterGrid(elevation=cfg1.grid.elevation)
    for backend in ("rbpg", "fista", "ista"):
        xs, hists, its, sts = [], [], [], []
        orders, supports, amps, scores = [], [], [], []
        for p in range(npx):
            sc = T.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=int(pseeds[p]))
            obj = T.Objective(dictionary=a, measurement=pix[p].astype(np.complex128), lambda_reg=float(lam[p]))
            sol = {"rbpg": T.rbpg_solve, "fista": T.fista_solve, "ista": T.ista_solve}[backend](obj, sc)
            xs.append(sol.x_hat)
            h = np.full(501, np.nan)
            h[: sol.objective_history.size] = sol.objective_history
            hists.append(h)
            its.append(sol.iterations_used)
            sts.append(STATUS[sol.status.value])
            est = T.slimmer_pipeline(obj, grid, T.PipelineConfig(solver=sc, backend=backend, k_max=2))
            orders.append(est.model_order)
            s = np.full(2, -1)
            s[: est.support.size] = est.support
            supports.append(s)
            am = np.zeros(2, dtype=complex)
            am[: est.amplitudes.size] = est.amplitudes
            amps.append(am)
            sv = np.full(3, np.nan)
            sv[: est.selection_scores.size] = est.selection_scores
            scores.append(sv)
        put(f"cfg1/{backend}/x", np.array(xs))
        put(f"cfg1/{backend}/hist", np.array(hists))
        put(f"cfg1/{backend}/iters", np.array(its))
        put(f"cfg1/{backend}/status", np.array(sts))
        put(f"cfg1/{backend}/order", np.array(orders))
        put(f"cfg1/{backend}/support", np.array(supports))
        put(f"cfg1/{backend}/amps", np.array(amps))
        put(f"cfg1/{backend}/scores", np.array(scores))

    # --- solver edge cases (test_solver.py:185-247)
    eye = np.eye(6)
    bid = rand_c(rng, 6) * 2
    put("edge/eye_b", bid)
    for backend, fn in (("rbpg", T.rbpg_solve), ("fista", T.fista_solve), ("ista", T.ista_solve)):
        sol = fn(T.Objective(dictionary=eye, measurement=bid, lambda_reg=0.5), T.SolverConfig(num_blocks=2, max_iters=2000, tol=1e-12))
        put(f"edge/eye_{backend}_x", sol.x_hat)
        put(f"edge/eye_{backend}_iters", sol.iterations_used)
        sol = fn(T.Objective(dictionary=np.eye(4), measurement=np.zeros(4), lambda_reg=0.5), T.SolverConfig(num_blocks=2, max_iters=50))
        put(f"edge/zero_{backend}_status", STATUS[sol.status.value])
        put(f"edge/zero_{backend}_hist", sol.objective_history)
    obj = T.Objective(dictionary=a, measurement=pix[3].astype(np.complex128), lambda_reg=float(lam[3]))
    for backend, fn in (("rbpg", T.rbpg_solve), ("fista", T.fista_solve)):
        sol = fn(obj, T.SolverConfig(num_blocks=8, fixed_iters=37, tol=1e-1, seed=9))
        put(f"edge/fixed_{backend}_iters", sol.iterations_used)
        put(f"edge/fixed_{backend}_hist", sol.objective_history)
        put(f"edge/fixed_{backend}_status", STATUS[sol.status.value])
        sol = fn(obj, T.SolverConfig(num_blocks=8, max_iters=60, tol=1e-6, alpha_init_scale=4.0, seed=9))
        put(f"edge/scale4_{backend}_x", sol.x_hat)
        put(f"edge/scale4_{backend}_hist", sol.objective_history)
        sol = fn(obj, T.SolverConfig(num_blocks=8, max_iters=60, tol=1e-6, alpha_init_scale=1e30, c_alpha=0.999999, seed=9))
        put(f"edge/lsfail_{backend}_status", STATUS[sol.status.value])
        put(f"edge/lsfail_{backend}_iters", sol.iterations_used)
        put(f"edge/lsfail_{backend}_hist", sol.objective_history)

    # --- slimmer.py: detect_support fixtures (test_slimmer.py:36-78) and model selection
    ds = []
    g10 = T.ParameterGrid.uniform((0, 9), 10)
    x = np.zeros(10, dtype=complex)
    x[4] = 2 - 1j
    ds.append((x, (10,), 3))
    x = np.zeros(20)
    x[[5, 6, 14, 2, 17]] = [1.0, 0.4, 0.8, 0.08, 0.07]
    ds.append((x, (20,), 2))
    x = np.zeros(10)
    x[[3, 8]] = [1.0, 1e-12]
    ds.append((x, (10,), 2))
    x = np.zeros(15)
    x[5] = 1.0
    x[9] = 0.6
    ds.append((x, (5, 3), 2))
    x = np.zeros(10)
    x[[1, 4, 7]] = [0.5, 1.0, 0.8]
    ds.append((x, (10,), 2))
    ds.append((np.zeros(10), (10,), 2))
    for i in range(6):
        ds.append((rand_c(rng, 60) * (rng.random(60) < 0.3), (60,), 3))
        ds.append((rand_c(rng, 4 * 5 * 3) * (rng.random(60) < 0.2), (4, 5, 3), 3))
    for i, (x, shape, k) in enumerate(ds):
        if len(shape) == 1:
            gr = T.ParameterGrid.uniform((0, shape[0] - 1), shape[0])
        else:
            gr = T.ParameterGrid.uniform((0, shape[0] - 1), shape[0], tuple(("linear", 0, 1, c) for c in shape[1:2]) + tuple(("seasonal", 0, 1, c) for c in shape[2:3]))
        put(f"detect{i}/x", x)
        put(f"detect{i}/shape", np.array(shape))
        put(f"detect{i}/k", k)
        put(f"detect{i}/out", T.detect_support(x, gr, k))
    put("detect/count", len(ds))
    _ = g10
    dup = np.array([[1.0, 1.0, 0.0], [0.0, 0.0, 1.0]], dtype=complex)
    k_hat, sup, sc = T.model_select(T.Objective(dictionary=dup, measurement=np.array([1.0, 0.5]), lambda_reg=0.0), np.array([0, 1, 2]), 3)
    put("msel_dup/k", k_hat)
    put("msel_dup/support", sup)
    put("msel_dup/scores", sc)

    # --- model.py: steering dictionary with two motion axes (model.py:254-323)
    geom = T.demo_geometry(n_acquisitions=29, seed=7)
    sgrid = T.ParameterGrid.uniform((-20.0, 20.0), 11, (("linear", -0.02, 0.02, 3), ("seasonal", 0.0, 0.01, 2)))
    put("steer/xi", T.spatial_frequencies(geom))
    put("steer/eta", T.temporal_frequencies(geom, sgrid.motion_bases))
    put("steer/elev", sgrid.elevation)
    put("steer/ax0", sgrid.motion_axes[0])
    put("steer/ax1", sgrid.motion_axes[1])
    put("steer/a", T.build_steering_matrix(geom, sgrid).entries)

    # --- svd_wiener backend (solver.py:393-407, slimmer.py:198-199)
    for mu in (0.0, 2.5):
        xs, orders, sups = [], [], []
        for p in range(npx):
            obj = T.Objective(dictionary=a, measurement=pix[p].astype(np.complex128), lambda_reg=0.0)
            xs.append(T.svd_wiener_solve(obj, mu))
            est = T.slimmer_pipeline(obj, grid, T.PipelineConfig(backend="svd_wiener", wiener_mu=mu, k_max=2))
            orders.append(est.model_order)
            sp = np.full(2, -1)
            sp[: est.support.size] = est.support
            sups.append(sp)
        put(f"wiener{mu}/x", np.array(xs))
        put(f"wiener{mu}/order", np.array(orders))
        put(f"wiener{mu}/support", np.array(sups))

    # --- cli.py solve on a TSTK1 stack (the production caller, cli.py:112-174)
    import json
    import tempfile

    from tomobpdn import cli, simulate, stack

    sgeom = T.demo_geometry(n_acquisitions=29, seed=3)
    rho = sgeom.rayleigh_resolution
    prng = substream(99, 1)
    rows = []
    for p in range(24):
        k = p % 3
        scs = tuple(simulate.Scatterer(elevation=float(prng.uniform(-2 * rho, 2 * rho)), amplitude=float(prng.uniform(0.6, 1.4)), phase=float(prng.uniform(0, 6.28))) for _ in range(k))
        sc = simulate.Scenario(geometry=sgeom, scatterers=scs, snr_db=tuple(10.0 for _ in scs), seed=p)
        rows.append(simulate.synthesize_pixel(sc, substream(99, 100 + p)))
    rows.append(np.zeros(29))
    with tempfile.TemporaryDirectory() as td:
        spath = os.path.join(td, "s.tstk")
        stack.write_stack(spath, sgeom, np.array(rows))
        put("cli/stack", np.frombuffer(open(spath, "rb").read(), dtype=np.uint8))
        cfgp = os.path.join(td, "c.json")
        open(cfgp, "w").write(json.dumps({"max_iters": 500, "tol": 1e-6, "seed": 77}))
        put("cli/config", json.dumps({"max_iters": 500, "tol": 1e-6, "seed": 77}))
        grids = {
            "g1": {"elevation": {"min": -2 * rho, "max": 2 * rho, "count": 81}},
            "g2": {"elevation": {"min": -2 * rho, "max": 2 * rho, "count": 41}, "motion": [{"base": "linear", "min": -0.01, "max": 0.01, "count": 5}]},
        }
        for gname, gd in grids.items():
            put(f"cli/{gname}", json.dumps(gd))
            gp = os.path.join(td, gname + ".json")
            open(gp, "w").write(json.dumps(gd))
            for backend in (("rbpg", "fista") if gname == "g1" else ("rbpg",)):
                op = os.path.join(td, f"{gname}_{backend}.jsonl")
                assert cli.main(["solve", "--stack", spath, "--grid", gp, "--out", op, "--config", cfgp, "--backend", backend, "--csv", op + ".csv"]) == 0
                put(f"cli/{gname}_{backend}_jsonl", open(op).read())

    path = os.path.join(os.path.dirname(__file__), "golden_v1.npz")
    np.savez_compressed(path, **OUT)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(OUT)} arrays)")


if __name__ == "__main__":
    main()
