"""Batched Monte-Carlo detection harness ("next" row 3).

Mirrors the reference ``simulate.py`` API: ``Scatterer`` (simulate.py:34-50), ``Scenario``
(:53-138), ``demo_geometry`` (:152-178), ``separation_unit`` (:181-191), ``synthesize_pixel``
(:194-205), ``detection_criterion`` (:208-234), ``DetectionResult`` (:237-246),
``wilson_interval`` (:249-259), ``MonteCarloSetup`` (:262-290), ``run_pipeline_realization``
(:297-338), ``monte_carlo_detection`` (:354-424), ``results_to_csv`` (:427-440).

What changes is the execution: the reference runs one full pipeline per realization in a process
pool; here every realization of every (kappa, SNR) cell is one pixel of a single device batch per
method (one shared dictionary, the batched solver and the fused selection kernel).  The
realizations themselves are drawn on the host exactly as the reference draws them (numpy Philox
substream keyed (scenario seed, cell * realizations + r); phase, ziggurat normals, nested solver
seed in the same order), so the synthesized pixels are bit-identical to the reference's and the
per-realization outcomes differ only where the float32 solve lands on the other side of a
detection decision.  ``draws="device"`` instead draws the realizations on the GPU
(``tb_synthesize_pairs``: the same Philox substreams, Box-Muller normals), so the whole sweep runs
on the device with statistically equivalent draws.
"""

from __future__ import annotations

import math
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from .exceptions import ConfigurationError
from .geometry import AcquisitionGeometry, steering_column, steering_dictionary
from .grid import ParameterGrid
from .solver import SolverConfig

_MASK64 = (1 << 64) - 1


def substream(seed: int, stream_id: int = 0) -> np.random.Generator:
    """numpy Philox generator keyed [seed, stream_id] (rng.py:17-24)."""
    return np.random.Generator(np.random.Philox(key=[int(seed) & _MASK64, int(stream_id) & _MASK64]))


def derive_seed(rng: np.random.Generator) -> int:
    """A 63-bit nested seed drawn from ``rng`` (rng.py:27-29)."""
    return int(rng.integers(0, 2**63 - 1))


@dataclass(frozen=True)
class Scatterer:
    elevation: float
    motion: tuple = ()
    amplitude: float = 1.0
    phase: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "motion", tuple(float(p) for p in self.motion))
        if not (np.isfinite(self.amplitude) and self.amplitude >= 0):
            raise ConfigurationError(f"amplitude must be >= 0, got {self.amplitude}")

    @property
    def gain(self) -> complex:
        return self.amplitude * np.exp(1j * self.phase)


@dataclass(frozen=True)
class Scenario:
    geometry: AcquisitionGeometry
    scatterers: tuple = ()
    snr_db: tuple = ()
    motion_bases: tuple = ()
    realizations: int = 1
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "scatterers", tuple(self.scatterers))
        object.__setattr__(self, "snr_db", tuple(float(v) for v in self.snr_db))
        object.__setattr__(self, "motion_bases", tuple(self.motion_bases))
        if len(self.snr_db) != len(self.scatterers):
            raise ConfigurationError("snr_db list must match scatterer count")
        if any(len(sc.motion) != len(self.motion_bases) for sc in self.scatterers):
            raise ConfigurationError("scatterer motion values must match motion_bases length")
        if self.realizations < 1:
            raise ConfigurationError("realizations must be >= 1")

    @property
    def noise_variance(self) -> float:
        if not self.scatterers:
            return 0.0
        ref = self.scatterers[0]
        return ref.amplitude**2 * 10.0 ** (-self.snr_db[0] / 10.0)


def demo_geometry(n_acquisitions: int = 29, aperture: float = 270.0, wavelength: float = 0.031, slant_range: float = 6.2e5,
                  time_span: float = 2.0, jitter: float = 0.35, seed: int = 12345) -> AcquisitionGeometry:
    """Jittered, irregular baseline stack (simulate.py:152-178)."""
    rng = substream(seed, 2)
    b = np.linspace(-0.5, 0.5, n_acquisitions) + rng.uniform(-jitter, jitter, n_acquisitions) / (n_acquisitions - 1)
    b = np.sort(b)
    b = (b - b.min()) / (b.max() - b.min()) - 0.5
    t = np.sort(rng.uniform(0.0, time_span, n_acquisitions))
    return AcquisitionGeometry(baselines=b * aperture, times=t, wavelength=wavelength, slant_range=slant_range)


def separation_unit(geometry: AcquisitionGeometry) -> float:
    """First null of the sampled point response: half the nominal Rayleigh resolution."""
    return geometry.rayleigh_resolution / 2.0


def synthesize_pixel(scenario: Scenario, rng: np.random.Generator) -> np.ndarray:
    """g = sum_k gain_k a(s_k, p_k) + sqrt(sigma^2/2) (n_re + j n_im), complex128 (simulate.py:194-205)."""
    geom = scenario.geometry
    g = np.zeros(geom.n_acquisitions, dtype=complex)
    for sc in scenario.scatterers:
        g += sc.gain * steering_column(geom, sc.elevation, sc.motion, scenario.motion_bases)
    sigma2 = scenario.noise_variance
    if sigma2 > 0.0:
        scale = math.sqrt(sigma2 / 2.0)
        noise = rng.standard_normal(g.size) + 1j * rng.standard_normal(g.size)
        g = g + scale * noise
    return g


def _match(elevations, truths, tol: float) -> bool:
    # greedy nearest-neighbour pairing, first minimum on ties (simulate.py:225-234)
    remaining = list(elevations)
    for s in truths:
        if not remaining:
            return False
        errors = [abs(e - s) for e in remaining]
        j = int(np.argmin(errors))
        if errors[j] > tol:
            return False
        remaining.pop(j)
    return True


def detection_criterion(estimates, truth: Scenario, tol: float | None = None) -> bool:
    """Correct model order and every true elevation matched within ``tol`` (simulate.py:208-234)."""
    if tol is None:
        tol = truth.geometry.rayleigh_resolution / 4.0
    if tol <= 0:
        raise ConfigurationError(f"tol must be > 0, got {tol}")
    truths = [sc.elevation for sc in truth.scatterers]
    if estimates.model_order != len(truths):
        return False
    return _match(estimates.elevations, truths, tol)


@dataclass(frozen=True)
class DetectionResult:
    kappa: float
    snr_db: float
    method: str
    p_d: float
    realizations: int
    ci_low: float
    ci_high: float


def wilson_interval(successes: int, total: int, z: float = 1.959964) -> tuple:
    """95% Wilson score interval (simulate.py:249-259)."""
    if total <= 0:
        raise ConfigurationError("total must be > 0")
    p = successes / total
    z2 = z * z
    denom = 1.0 + z2 / total
    center = (p + z2 / (2 * total)) / denom
    half = z * math.sqrt(p * (1 - p) / total + z2 / (4 * total * total)) / denom
    return max(0.0, center - half), min(1.0, center + half)


@dataclass(frozen=True)
class MonteCarloSetup:
    grid_size: int = 161
    grid_halfspan: float = 4.0
    tol_factor: float = 0.3
    delta_phi: float | None = 0.0
    k_max: int = 2
    solver: SolverConfig = field(default_factory=SolverConfig)

    def __post_init__(self):
        if self.grid_size < 3:
            raise ConfigurationError("grid_size must be >= 3")
        if self.grid_halfspan <= 0 or self.tol_factor <= 0:
            raise ConfigurationError("grid_halfspan and tol_factor must be > 0")


def harness_grid(base: Scenario, setup: MonteCarloSetup) -> ParameterGrid:
    unit = separation_unit(base.geometry)
    return ParameterGrid.uniform((-setup.grid_halfspan * unit, setup.grid_halfspan * unit), setup.grid_size)


def _snap(grid: ParameterGrid, value: float) -> float:
    return float(grid.elevation[np.argmin(np.abs(grid.elevation - value))])


def _truth(base: Scenario, grid: ParameterGrid, kappa: float, snr: float, dphi: float) -> Scenario:
    half_sep = kappa * separation_unit(base.geometry) / 2.0
    return replace(base, scatterers=(Scatterer(elevation=_snap(grid, -half_sep), amplitude=1.0, phase=0.0),
                                     Scatterer(elevation=_snap(grid, +half_sep), amplitude=1.0, phase=dphi)),
                   snr_db=(snr, snr), motion_bases=())


def draw_realization(base: Scenario, grid: ParameterGrid, kappa: float, snr: float, setup: MonteCarloSetup, stream_id: int):
    """(pixel complex128 [n], nested solver seed, truth Scenario) in the reference's draw order
    (simulate.py:309-329): phase (when drawn), the two normal vectors, then derive_seed."""
    rng = substream(base.seed, stream_id)
    dphi = float(rng.uniform(0.0, 2.0 * np.pi)) if setup.delta_phi is None else setup.delta_phi
    truth = _truth(base, grid, kappa, snr, dphi)
    g = synthesize_pixel(truth, rng)
    return g, derive_seed(rng), truth


def _draw_chunk(args):
    base, grid, setup, items = args
    out = []
    for kappa, snr, sid in items:
        g, seed, truth = draw_realization(base, grid, kappa, snr, setup, sid)
        out.append((g, seed, [sc.elevation for sc in truth.scatterers]))
    return out


def _draw_all(base, grid, setup, items, workers: int):
    if workers <= 1 or len(items) < 2048:
        return _draw_chunk((base, grid, setup, items))
    step = (len(items) + 4 * workers - 1) // (4 * workers)
    chunks = [(base, grid, setup, items[i:i + step]) for i in range(0, len(items), step)]
    with ProcessPoolExecutor(max_workers=workers) as pool:
        return [r for part in pool.map(_draw_chunk, chunks) for r in part]


def monte_carlo_outcomes(base: Scenario, kappas, snrs, methods, realizations: int, setup: MonteCarloSetup | None = None,
                         workers: int = 1, device=None, draws: str = "host"):
    """Per-realization detection outcomes, cells in the reference's (kappa, snr, method) order.

    ``draws`` "host": every realization drawn on the host exactly as the reference draws it
    (bit-identical pixels and nested seeds).  "device": drawn by the synthesis kernel
    (``Dictionary.synthesize_pairs``) from the same Philox substreams with Box-Muller normals --
    statistically equivalent, and the whole harness then runs on the GPU.
    Returns (cells, outcomes) with outcomes a bool array [len(cells), realizations].
    """
    from .slimmer import PipelineConfig, pipeline_batch
    from .solver import Dictionary

    if realizations < 1:
        raise ConfigurationError("realizations must be >= 1")
    setup = setup or MonteCarloSetup()
    for meth in methods:
        if meth not in ("rbpg", "ista", "fista", "svd_wiener"):
            raise ConfigurationError(f"unknown backend {meth!r}")
    grid = harness_grid(base, setup)
    unit = separation_unit(base.geometry)
    tol = setup.tol_factor * unit
    if draws not in ("host", "device"):
        raise ConfigurationError(f"draws must be 'host' or 'device', got {draws!r}")
    cells = [(k, s, meth) for k in kappas for s in snrs for meth in methods]
    items = [(cells[c][0], cells[c][1], c * realizations + r) for c in range(len(cells)) for r in range(realizations)]
    d = Dictionary(steering_dictionary(base.geometry, grid, device=device))
    if draws == "host":
        drawn = _draw_all(base, grid, setup, items, workers)
        pixels = np.stack([d_[0] for d_ in drawn]).astype(np.complex64)
        seeds = np.array([d_[1] for d_ in drawn], dtype=np.uint64)
        truths = [d_[2] for d_ in drawn]
    else:
        # the two scatterers at the grid points nearest -/+ kappa unit / 2, unit amplitude, phases 0
        # and delta_phi (drawn when None), noise variance from the first scatterer (simulate.py:309-329)
        elev = np.asarray(grid.elevation, dtype=float)
        unit_half = np.array([it[0] for it in items]) * unit / 2.0
        c0 = np.abs(elev[None, :] + unit_half[:, None]).argmin(axis=1)
        c1 = np.abs(elev[None, :] - unit_half[:, None]).argmin(axis=1)
        phase = np.full(len(items), np.nan if setup.delta_phi is None else setup.delta_phi, dtype=np.float32)
        sigma = np.sqrt(10.0 ** (-np.array([it[1] for it in items]) / 10.0)).astype(np.float32)
        pixels, seeds = d.synthesize_pairs(base.seed, [it[2] for it in items], c0, c1, phase, sigma)
        seeds = seeds.view(torch_int64())  # CUDA gathers do not take uint64; solve() reinterprets int64 seeds
        truths = [[float(elev[a]), float(elev[b])] for a, b in zip(c0, c1)]
    outcomes = np.zeros(len(items), dtype=bool)
    for meth in dict.fromkeys(methods):
        rows = np.array([i for i in range(len(items)) if cells[i // realizations][2] == meth])
        # svd_wiener: mu = noise variance * L depends on the cell's SNR (simulate.py:330)
        mus = np.array([10.0 ** (-cells[i // realizations][1] / 10.0) * grid.flat_size if meth == "svd_wiener" else 0.0 for i in rows])
        for mu in np.unique(mus):
            grp = rows[mus == mu]
            cfg = PipelineConfig(solver=setup.solver, backend=meth, k_max=setup.k_max, wiener_mu=float(mu))
            sel = grp if draws == "host" else _torch_index(grp, pixels.device)
            est = pipeline_batch(d, pixels[sel], grid, cfg, seeds=seeds[sel] if meth == "rbpg" else None)
            order = est.model_order.cpu().numpy()
            elev = est.elevations.cpu().numpy()
            err = est.error.cpu().numpy()
            for j, i in enumerate(grp):
                ok = not err[j] and order[j] == len(truths[i]) and _match(elev[j, : order[j]], truths[i], tol)
                outcomes[i] = ok
    return cells, outcomes.reshape(len(cells), realizations)


def torch_int64():
    import torch

    return torch.int64


def _torch_index(rows, device):
    import torch

    return torch.as_tensor(np.asarray(rows, dtype=np.int64), device=device)


def monte_carlo_detection(base: Scenario, kappas, snrs, methods, realizations: int, setup: MonteCarloSetup | None = None,
                          workers: int = 1, device=None, draws: str = "host") -> list:
    """Detection rate per (kappa, SNR, method) cell with Wilson 95% CIs (simulate.py:354-424)."""
    cells, outcomes = monte_carlo_outcomes(base, kappas, snrs, methods, realizations, setup, workers, device, draws)
    out = []
    for (kappa, snr, meth), hits in zip(cells, outcomes):
        h = int(hits.sum())
        lo, hi = wilson_interval(h, realizations)
        out.append(DetectionResult(kappa=kappa, snr_db=snr, method=meth, p_d=h / realizations, realizations=realizations,
                                   ci_low=lo, ci_high=hi))
    return out


def run_pipeline_realization(base: Scenario, dictionary, grid: ParameterGrid, kappa: float, snr: float, method: str,
                             setup: MonteCarloSetup, tol: float, stream_id: int) -> bool:
    """One realization through the batched path (simulate.py:297-338)."""
    from .slimmer import PipelineConfig, pipeline_batch

    g, seed, truth = draw_realization(base, grid, kappa, snr, setup, stream_id)
    mu = truth.noise_variance * grid.flat_size
    cfg = PipelineConfig(solver=replace(setup.solver, seed=seed), backend=method, k_max=setup.k_max, wiener_mu=mu)
    est = pipeline_batch(dictionary, g.astype(np.complex64).reshape(1, -1), grid, cfg,
                         seeds=np.array([seed], dtype=np.uint64) if method == "rbpg" else None)
    if int(est.error[0].item()):
        return False
    return detection_criterion(est.estimates(0), truth, tol)


def results_to_csv(results, path) -> None:
    """kappa,snr_db,method,p_d,ci_low,ci_high,n (simulate.py:427-440)."""
    import csv

    with open(Path(path), "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["kappa", "snr_db", "method", "p_d", "ci_low", "ci_high", "n"])
        for r in results:
            w.writerow([repr(r.kappa), repr(r.snr_db), r.method, repr(r.p_d), repr(r.ci_low), repr(r.ci_high), r.realizations])

