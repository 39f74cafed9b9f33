"""Acquisition geometry and exact steering vectors (host side of the Monte-Carlo harness).

Mirrors the reference ``model.py``: ``AcquisitionGeometry`` (model.py:38-124, same fields and
validation), ``spatial_frequencies`` xi_n = 2 b_n / (lambda r) (model.py:254-259),
``temporal_frequencies`` eta_{m,n} = 2 tau_m(t_n) / lambda (model.py:262-277),
``steering_column`` (model.py:280-293) and ``rayleigh_resolution`` (model.py:326-335).  These are
O(n) host computations feeding the batched device path; the dense dictionary is built on the
device by ``grid.build_steering_matrix``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import ConfigurationError, GeometryError

_GEOMETRY_KEYS = {"baselines_m", "times_yr", "wavelength_m", "range_m"}


def _tau(name: str, t: np.ndarray) -> np.ndarray:
    # motion base functions, model.py:27-30
    if name == "linear":
        return t
    if name == "seasonal":
        return np.sin(2.0 * np.pi * t)
    raise ConfigurationError(f"unknown base function {name!r}; known: ['linear', 'seasonal']")


def _positive(name: str, value: float) -> None:
    if not (np.isfinite(value) and value > 0):
        raise GeometryError(f"{name} must be > 0, got {value}")


@dataclass(frozen=True, eq=False)
class AcquisitionGeometry:
    """Perpendicular baselines b_n [m], times t_n [yr], wavelength [m], slant range [m]."""

    baselines: np.ndarray
    times: np.ndarray
    wavelength: float
    slant_range: float

    def __post_init__(self):
        b = np.asarray(self.baselines, dtype=float)
        t = np.asarray(self.times, dtype=float)
        object.__setattr__(self, "baselines", b)
        object.__setattr__(self, "times", t)
        if b.ndim != 1 or t.ndim != 1 or b.size != t.size:
            raise GeometryError("baselines and times must be 1-d with equal length")
        if b.size < 2:
            raise GeometryError("need at least 2 acquisitions")
        if not (np.isfinite(b).all() and np.isfinite(t).all()):
            raise GeometryError("baselines/times must be finite")
        _positive("wavelength", self.wavelength)
        _positive("slant range", self.slant_range)
        if self.aperture <= 0:
            raise GeometryError("aperture extent max(b) - min(b) must be > 0")
        b.setflags(write=False)
        t.setflags(write=False)

    def __eq__(self, other):
        if not isinstance(other, AcquisitionGeometry):
            return NotImplemented
        return (np.array_equal(self.baselines, other.baselines) and np.array_equal(self.times, other.times)
                and self.wavelength == other.wavelength and self.slant_range == other.slant_range)

    @property
    def n_acquisitions(self) -> int:
        return int(self.baselines.size)

    @property
    def aperture(self) -> float:
        return float(self.baselines.max() - self.baselines.min())

    @property
    def rayleigh_resolution(self) -> float:
        return rayleigh_resolution(self.wavelength, self.slant_range, self.aperture)

    def to_dict(self) -> dict:
        return {"baselines_m": self.baselines.tolist(), "times_yr": self.times.tolist(),
                "wavelength_m": self.wavelength, "range_m": self.slant_range}

    @classmethod
    def from_dict(cls, data: dict) -> "AcquisitionGeometry":
        if not isinstance(data, dict):
            raise GeometryError("geometry must be a JSON object")
        keys = set(data)
        if keys - _GEOMETRY_KEYS:
            raise GeometryError(f"unknown geometry keys: {sorted(keys - _GEOMETRY_KEYS)}")
        if _GEOMETRY_KEYS - keys:
            raise GeometryError(f"missing geometry keys: {sorted(_GEOMETRY_KEYS - keys)}")
        return cls(np.asarray(data["baselines_m"], dtype=float), np.asarray(data["times_yr"], dtype=float),
                   float(data["wavelength_m"]), float(data["range_m"]))


def rayleigh_resolution(wavelength: float, slant_range: float, aperture: float) -> float:
    """rho_s = lambda r / delta_b."""
    _positive("wavelength", wavelength)
    _positive("slant_range", slant_range)
    _positive("aperture", aperture)
    return wavelength * slant_range / aperture


def spatial_frequencies(geom: AcquisitionGeometry) -> np.ndarray:
    xi = 2.0 * geom.baselines / (geom.wavelength * geom.slant_range)
    if not np.isfinite(xi).all():
        raise GeometryError("non-finite spatial frequencies")
    return xi


def temporal_frequencies(geom: AcquisitionGeometry, base_functions: tuple) -> np.ndarray:
    if not base_functions:
        return np.zeros((0, geom.n_acquisitions))
    return np.vstack([2.0 * _tau(name, geom.times) / geom.wavelength for name in base_functions])


def steering_column(geom: AcquisitionGeometry, elevation: float, motion: tuple = (), motion_bases: tuple = ()) -> np.ndarray:
    """Exact (off-grid capable) steering vector exp(2 pi j (xi s + eta . p)), complex128."""
    if len(motion) != len(motion_bases):
        raise ConfigurationError("motion values and base functions must pair up")
    phase = spatial_frequencies(geom) * elevation
    if motion:
        phase = phase + temporal_frequencies(geom, tuple(motion_bases)).T @ np.asarray(motion, dtype=float)
    return np.exp(2j * np.pi * phase)


def steering_dictionary(geom: AcquisitionGeometry, grid, device=None):
    """The dense dictionary of ``geom`` over ``grid`` (model.py:296-323), built on the device."""
    from .grid import build_steering_matrix

    eta = temporal_frequencies(geom, grid.motion_bases) if grid.motion_axes else None
    return build_steering_matrix(spatial_frequencies(geom), grid, eta=eta, sign=1.0, device=device)
