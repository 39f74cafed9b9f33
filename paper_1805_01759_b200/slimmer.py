"""SL1MMER pipeline mirrored from the reference ``slimmer.py``, on the device.

``PipelineConfig`` (slimmer.py:31-52), ``ScattererEstimates`` (:55-74), ``slimmer_pipeline``
(:193-212), ``build_objective`` (:215-222), ``estimates_to_record`` (:225-234) keep the
reference names and layouts.  ``pipeline_batch`` is the batched production entry: lambda rule,
per-pixel seed rule (cli.py:102), solve, and the fused detect_support -> model_select ->
estimate_params kernel, all on one stream with no host round trip between stages.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .exceptions import ConfigurationError, EstimationError
from .grid import ParameterGrid
from .prox import Objective, default_lambda
from .solver import BatchSolution, Dictionary, SolverConfig, _torch, dictionary_for

BACKENDS = ("rbpg", "ista", "fista", "svd_wiener")  # slimmer.py:25
PEAK_FLOOR = 1e-8  # slimmer.py:28


@dataclass(frozen=True)
class PipelineConfig:
    """Per-pixel pipeline settings: solver, backend choice, model order cap."""

    solver: SolverConfig = field(default_factory=SolverConfig)
    backend: str = "rbpg"
    k_max: int = 2
    wiener_mu: float = 0.0

    def __post_init__(self):
        if self.backend not in BACKENDS:
            raise ConfigurationError(f"unknown backend {self.backend!r}; known: {BACKENDS}")
        if self.k_max < 1:
            raise ConfigurationError(f"k_max must be >= 1, got {self.k_max}")
        if not (np.isfinite(self.wiener_mu) and self.wiener_mu >= 0):
            raise ConfigurationError(f"wiener_mu must be >= 0, got {self.wiener_mu}")


@dataclass(frozen=True)
class ScattererEstimates:
    """Model order, per-scatterer parameters, and selection telemetry."""

    model_order: int
    elevations: np.ndarray
    motion_params: np.ndarray
    amplitudes: np.ndarray
    selection_scores: np.ndarray
    support: np.ndarray

    def __post_init__(self):
        k = self.model_order
        if not (self.elevations.shape[0] == k and self.amplitudes.shape[0] == k and self.motion_params.shape[0] == k and self.support.shape[0] == k):
            raise EstimationError("per-scatterer vectors must have length model_order")


@dataclass
class BatchEstimates:
    """Device outputs of ``pipeline_batch`` (one row per pixel, k_max columns, -1/0 padded)."""

    model_order: object  # int32 [P]
    support: object  # int64 [P, k_max]
    amplitudes: object  # complex128 [P, k_max]
    elevations: object  # float64 [P, k_max]
    motion_params: object  # float64 [P, k_max, n_axes]
    selection_scores: object  # float64 [P, k_max + 1] (NaN padded)
    n_scores: object  # int32 [P]
    error: object  # int32 [P]
    solution: BatchSolution | None = None
    lam: object = None

    def estimates(self, i: int) -> ScattererEstimates:
        k = int(self.model_order[i].item())
        if int(self.error[i].item()):
            raise EstimationError("support columns are rank deficient")
        ns = int(self.n_scores[i].item())
        return ScattererEstimates(
            model_order=k,
            elevations=self.elevations[i, :k].cpu().numpy(),
            motion_params=self.motion_params[i, :k].cpu().numpy(),
            amplitudes=self.amplitudes[i, :k].cpu().numpy(),
            selection_scores=self.selection_scores[i, :ns].cpu().numpy(),
            support=self.support[i, :k].cpu().numpy().astype(int),
        )


class _GridDev:
    """Grid description uploaded once per (grid, device)."""

    def __init__(self, grid: ParameterGrid, device):
        torch = _torch()
        self.n_elev = int(grid.elevation.size)
        self.n_axes = len(grid.motion_axes)
        self.sizes = (ctypes.c_int32 * max(1, self.n_axes))(*([a.size for a in grid.motion_axes] or [1]))
        self.elev = torch.from_numpy(np.array(grid.elevation, dtype=np.float64)).to(device)
        mot = np.concatenate([np.asarray(a, dtype=np.float64) for a in grid.motion_axes]) if self.n_axes else np.zeros(1)
        self.motion = torch.from_numpy(mot).to(device)


def _grid_dev(d: Dictionary, grid: ParameterGrid) -> _GridDev:
    """Device copy of the grid axes, cached on the dictionary: a pageable host->device copy per
    call would block the host behind the solver kernel already queued on the stream."""
    cache = d.__dict__.setdefault("_grid_cache", {})
    key = (np.asarray(grid.elevation, dtype=np.float64).tobytes(), tuple(np.asarray(a, dtype=np.float64).tobytes() for a in grid.motion_axes))
    g = cache.get(key)
    if g is None:
        g = cache[key] = _GridDev(grid, d.device)
    return g


def select_batch(d: Dictionary, x_hat, pixels, grid: ParameterGrid, k_max: int, params_per_scatterer: int | None = None) -> BatchEstimates:
    """detect_support -> model_select -> estimate_params for every pixel (slimmer.py:77-190)."""
    torch = _torch()
    if k_max < 1:
        raise ConfigurationError(f"k_max must be >= 1, got {k_max}")
    if grid.flat_size != d.m:
        raise ConfigurationError(f"grid has {grid.flat_size} nodes but the dictionary has {d.m} columns")
    b = d._pixels(pixels)
    p = int(b.shape[0])
    ppsc = 3 + len(grid.motion_axes) if params_per_scatterer is None else int(params_per_scatterer)
    g = _grid_dev(d, grid)
    dev = d.device
    order = torch.empty(p, dtype=torch.int32, device=dev)
    support = torch.empty((p, k_max), dtype=torch.int64, device=dev)
    amps = torch.empty((p, k_max), dtype=torch.complex128, device=dev)
    elevs = torch.empty((p, k_max), dtype=torch.float64, device=dev)
    motion = torch.empty((p, k_max, max(1, g.n_axes)), dtype=torch.float64, device=dev)
    scores = torch.empty((p, k_max + 1), dtype=torch.float64, device=dev)
    nsc = torch.empty(p, dtype=torch.int32, device=dev)
    err = torch.empty(p, dtype=torch.int32, device=dev)
    xt = x_hat.to(device=dev, dtype=torch.complex64).contiguous()
    with torch.cuda.device(dev):
        _lib.check(
            d._lib.tb_select(
                d.handle, _lib.ptr(xt), _lib.ptr(b), p, g.n_elev, g.n_axes, g.sizes, _lib.ptr(g.elev), _lib.ptr(g.motion),
                int(k_max), ppsc, _lib.ptr(order), _lib.ptr(support), _lib.ptr(amps), _lib.ptr(elevs), _lib.ptr(motion),
                _lib.ptr(scores), _lib.ptr(nsc), _lib.ptr(err), d._stream(),
            )
        )
    return BatchEstimates(order, support, amps, elevs, motion[:, :, : g.n_axes], scores, nsc, err)


def pipeline_batch(dictionary, pixels, grid: ParameterGrid, config: PipelineConfig, lam=None, beta: float = 0.05,
                   seeds=None, run_seed: int | None = None, first_pixel_id: int = 0, device=None) -> BatchEstimates:
    """The batched ``tomobpdn solve`` path: lambda, seeds, solve, selection on one stream.

    ``lam`` None selects beta * max|A^H b| per pixel (the reference default beta is 0.05,
    prox.py:153; BASELINE uses 0.1).  RBPG seeds default to the CLI rule
    derive_seed(substream(run_seed, first_pixel_id + i)) with run_seed = config.solver.seed
    (cli.py:102, 125).
    """
    d = dictionary if isinstance(dictionary, Dictionary) else Dictionary(dictionary, device=device)
    b = d._pixels(pixels)
    if config.backend == "svd_wiener":  # slimmer.py:198-199: linear estimator, then the same selection
        est = select_batch(d, d.wiener(b, config.wiener_mu), b, grid, config.k_max)
        return est
    p = int(b.shape[0])
    if lam is None:
        lam_t = d.default_lambda(b, beta) if config.solver.lambda_reg is None else None
        if lam_t is None:
            lam_t = np.full(p, float(config.solver.lambda_reg), dtype=np.float64)
    else:
        lam_t = lam
    if config.backend == "rbpg" and seeds is None:
        seeds = d.derive_seeds(config.solver.seed if run_seed is None else run_seed, p, first_pixel_id)
    sol = d.solve(b, lam_t, config.solver, config.backend, seeds=seeds)
    est = select_batch(d, sol.x_hat, b, grid, config.k_max)
    est.solution = sol
    est.lam = lam_t
    return est


def slimmer_pipeline(obj: Objective, grid: ParameterGrid, config: PipelineConfig) -> ScattererEstimates:
    """Run sparse solve, model selection, and debiasing for one pixel (slimmer.py:193-212)."""
    d = dictionary_for(obj.dictionary)
    if config.backend == "svd_wiener":
        return select_batch(d, d.wiener(obj.measurement.reshape(1, -1), config.wiener_mu), obj.measurement.reshape(1, -1), grid, config.k_max).estimates(0)
    seeds = np.array([int(config.solver.seed) & (2**64 - 1)], dtype=np.uint64) if config.backend == "rbpg" else None
    sol = d.solve(obj.measurement.reshape(1, -1), np.array([obj.lambda_reg]), config.solver, config.backend, seeds=seeds)
    est = select_batch(d, sol.x_hat, obj.measurement.reshape(1, -1), grid, config.k_max)
    return est.estimates(0)


def build_objective(dictionary, measurement, config: SolverConfig) -> Objective:
    """Assemble the L1LS instance, resolving the default lambda if unset (slimmer.py:215-222)."""
    lam = config.lambda_reg
    if lam is None:
        lam = default_lambda(dictionary, measurement)
    return Objective(dictionary=dictionary, measurement=measurement, lambda_reg=lam)


def estimates_to_record(pixel_id: int, est: ScattererEstimates) -> dict:
    """JSON-friendly record for one pixel, stable key order (slimmer.py:225-234)."""
    return {
        "pixel_id": pixel_id,
        "model_order": est.model_order,
        "elevations_m": [float(v) for v in est.elevations],
        "motion_params": [[float(v) for v in row] for row in est.motion_params],
        "amplitudes": [[float(a.real), float(a.imag)] for a in est.amplitudes],
        "support": [int(v) for v in est.support],
    }

