"""Install this package as the solve path of an imported reference ``tomobpdn``.

``install(tomobpdn)`` rebinds the reference's hot-path entry points -- ``solver.rbpg_solve``,
``solver.ista_solve``, ``solver.fista_solve`` (solver.py:250, 379, 384) and
``slimmer.slimmer_pipeline`` (slimmer.py:193) -- to adapters over this package, so the reference's
own callers run unmodified on the GPU: the CLI worker (cli.py:97-109 calls
``slimmer.slimmer_pipeline``), the bench loop (cli.py:284-302 builds its table from
``solver.*_solve``), the Monte-Carlo realization runner (simulate.py:297-335).  The adapters take
the reference's own objects (Objective, SolverConfig, ParameterGrid, PipelineConfig) and return the
reference's own result types (Solution, ScattererEstimates), field for field.  ``uninstall``
restores the originals.
"""

from __future__ import annotations

import numpy as np

from . import slimmer as _slimmer
from . import solver as _solver
from .grid import ParameterGrid
from .prox import Objective

_SAVED: dict = {}


def _objective(obj) -> Objective:
    return Objective(dictionary=np.asarray(obj.dictionary), measurement=np.asarray(obj.measurement), lambda_reg=float(obj.lambda_reg))


def _config(cfg) -> _solver.SolverConfig:
    return _solver.SolverConfig.from_dict(cfg.to_dict())


def _grid(grid) -> ParameterGrid:
    return ParameterGrid(elevation=grid.elevation, motion_axes=tuple(grid.motion_axes), motion_bases=tuple(grid.motion_bases))


def install(ref) -> None:
    """Rebind the reference module ``ref`` (the imported ``tomobpdn`` package) to this package."""
    rs, rl = ref.solver, ref.slimmer
    if _SAVED:
        return
    _SAVED.update(rbpg=rs.rbpg_solve, ista=rs.ista_solve, fista=rs.fista_solve, pipeline=rl.slimmer_pipeline)

    def solve_adapter(ours):
        def run(obj, config):
            sol = ours(_objective(obj), _config(config))
            return rs.Solution(
                x_hat=sol.x_hat, objective_history=sol.objective_history, iterations_used=sol.iterations_used,
                status=rs.SolverStatus(sol.status.value), wall_time=sol.wall_time,
            )

        return run

    def pipeline(obj, grid, config):
        pc = _slimmer.PipelineConfig(solver=_config(config.solver), backend=config.backend, k_max=config.k_max, wiener_mu=config.wiener_mu)
        est = _slimmer.slimmer_pipeline(_objective(obj), _grid(grid), pc)
        return rl.ScattererEstimates(
            model_order=est.model_order, elevations=est.elevations, motion_params=est.motion_params,
            amplitudes=est.amplitudes, selection_scores=est.selection_scores, support=est.support,
        )

    rs.rbpg_solve = solve_adapter(_solver.rbpg_solve)
    rs.ista_solve = solve_adapter(_solver.ista_solve)
    rs.fista_solve = solve_adapter(_solver.fista_solve)
    rl.slimmer_pipeline = pipeline


def uninstall(ref) -> None:
    """Restore the reference's own entry points."""
    if not _SAVED:
        return
    ref.solver.rbpg_solve = _SAVED["rbpg"]
    ref.solver.ista_solve = _SAVED["ista"]
    ref.solver.fista_solve = _SAVED["fista"]
    ref.slimmer.slimmer_pipeline = _SAVED["pipeline"]
    _SAVED.clear()
