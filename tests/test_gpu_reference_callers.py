"""The reference's OWN callers run unmodified on the drop-in ("callers to keep
working"): ``cli._solve_worker`` (cli.py:97-109), ``cli.cmd_bench`` (cli.py:274-362) and
``simulate.run_pipeline_realization`` (simulate.py:297-335), with the reference's
``slimmer.slimmer_pipeline`` / ``solver.*_solve`` rebound to this package by
``paper_1805_01759_b200.dropin.install`` -- the patch INTEGRATION.md §1 describes.  Each caller's
output is compared with the same caller on the reference's own CPU path in the same process.

Needs the unmodified reference importable (``baseline/_ref``, installed by the builder and shipped
with the repo snapshot); skipped with a reason otherwise.
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from oracle import reference_arm as R

    path = R.locate()
    if path is None:
        pytest.skip("unmodified reference not installed (baseline/_ref)")
    return R._import(path)


@pytest.fixture
def patched(ref):
    from paper_1805_01759_b200 import dropin

    dropin.install(ref)
    yield ref
    dropin.uninstall(ref)


def _cfg1(ref, npx):
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(1, num_pixels=npx)
    return batch.dictionary.astype(np.complex128), batch.pixels, ref.ParameterGrid(elevation=batch.grid.elevation)


@pytest.mark.parametrize("backend", ["rbpg", "fista"])
def test_cli_solve_worker(ref, backend):
    """cli._solve_worker: seed rule, build_objective (default lambda beta 0.05), slimmer_pipeline,
    estimates_to_record -- records identical to the reference's own worker."""
    from paper_1805_01759_b200 import dropin
    from tomobpdn import cli

    a, pix, grid = _cfg1(ref, 24)
    pc = ref.PipelineConfig(solver=ref.SolverConfig(max_iters=500, tol=1e-6), backend=backend, k_max=2)
    cli._solve_worker_init(a, grid, pc, 2018)
    want = [cli._solve_worker((i, pix[i].astype(complex))) for i in range(len(pix))]
    dropin.install(ref)
    try:
        got = [cli._solve_worker((i, pix[i].astype(complex))) for i in range(len(pix))]
    finally:
        dropin.uninstall(ref)
    for g, w in zip(got, want):
        assert g["pixel_id"] == w["pixel_id"]
        assert g["model_order"] == w["model_order"], (g, w)
        assert g["support"] == w["support"]
        assert g["elevations_m"] == w["elevations_m"]
        np.testing.assert_allclose(np.array(g["amplitudes"]).reshape(-1), np.array(w["amplitudes"]).reshape(-1), rtol=1e-5, atol=1e-7)


def test_cli_bench(ref, tmp_path):
    """cli.cmd_bench through cli.main: the report's per-solver median iterations and final
    objectives from the drop-in solvers equal the reference's."""
    from paper_1805_01759_b200 import dropin
    from tomobpdn import cli

    conf = tmp_path / "bench.json"
    conf.write_text(json.dumps({"n_values": [29], "l_values": [100, 400], "solvers": ["rbpg", "ista", "fista"], "repeats": 2,
                                "max_iters": 3000, "block_sweep": [2, 8]}))
    reports = []
    for use_gpu in (False, True):
        out = tmp_path / f"r{int(use_gpu)}.json"
        if use_gpu:
            dropin.install(ref)
        try:
            assert cli.main(["bench", "--config", str(conf), "--out", str(out)]) == 0
        finally:
            if use_gpu:
                dropin.uninstall(ref)
        reports.append(json.loads(out.read_text()))
    cpu, gpu = reports
    assert [(r["solver"], r["l"]) for r in gpu["runs"]] == [(r["solver"], r["l"]) for r in cpu["runs"]]
    for g, c in zip(gpu["runs"], cpu["runs"]):
        assert g["median_iters"] == c["median_iters"], (g, c)
        assert g["median_final_objective"] == pytest.approx(c["median_final_objective"], rel=1e-6)
    assert len(gpu["rbpg_block_sweep"]) == len(cpu["rbpg_block_sweep"])


def test_simulate_run_pipeline_realization(ref):
    """simulate.run_pipeline_realization (the Monte-Carlo inner call): identical detection outcomes."""
    from paper_1805_01759_b200 import dropin
    from tomobpdn import simulate

    geom = simulate.demo_geometry(n_acquisitions=29, seed=3)
    rho = geom.rayleigh_resolution
    grid = ref.ParameterGrid.uniform((-2.0 * rho, 2.0 * rho), 161)
    a = ref.build_steering_matrix(geom, grid).entries
    base = simulate.Scenario(geometry=geom, scatterers=(simulate.Scatterer(elevation=0.0),), snr_db=(10.0,), seed=11)
    setup = simulate.MonteCarloSetup()
    tol = setup.tol_factor * simulate.separation_unit(geom)
    cells = [(k, s, m, i) for k in (0.6, 1.2) for s in (3.0, 10.0) for m in ("rbpg", "fista") for i in range(3)]

    def run():
        return [simulate.run_pipeline_realization(base, a, grid, k, s, m, setup, tol, 100 * j + i) for j, (k, s, m, i) in enumerate(cells)]

    want = run()
    dropin.install(ref)
    try:
        got = run()
    finally:
        dropin.uninstall(ref)
    assert got == want
