"""Parameter grid: the flat-index decode the selection stage needs.

Mirrors the reference ``ParameterGrid`` (``model.py:154-235``): the dictionary's flat column
index enumerates the grid row-major with elevation as the leading axis
(``model.py:158-160``), ``values_at`` decodes (elevation, motion coefficients)
(``model.py:203-208``) and ``elevation_profile`` collapses motion axes by max
(``model.py:210-215``).  Geometry/steering construction is out of scope (the dictionary is
an input to the hot path), so only the grid description and its decode live here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import ConfigurationError, GridError

MOTION_BASES = ("linear", "seasonal")  # model.py:27-30


def _check_axis(values: np.ndarray, name: str) -> None:
    # model.py:141-151
    if values.ndim != 1 or values.size == 0:
        raise GridError(f"{name} axis must be a non-empty 1-d vector")
    if not np.all(np.isfinite(values)):
        raise GridError(f"{name} axis must be finite")
    if values.size >= 2:
        steps = np.diff(values)
        if np.any(steps <= 0):
            raise GridError(f"{name} axis must be strictly increasing")
        if not np.allclose(steps, steps[0], rtol=1e-9, atol=0.0):
            raise GridError(f"{name} axis must be uniformly spaced")


@dataclass(frozen=True)
class ParameterGrid:
    """Cartesian search grid over elevation and motion coefficients."""

    elevation: np.ndarray
    motion_axes: tuple = ()
    motion_bases: tuple = ()

    def __post_init__(self):
        elev = np.asarray(self.elevation, dtype=float)
        axes = tuple(np.asarray(a, dtype=float) for a in self.motion_axes)
        object.__setattr__(self, "elevation", elev)
        object.__setattr__(self, "motion_axes", axes)
        object.__setattr__(self, "motion_bases", tuple(self.motion_bases))
        _check_axis(elev, "elevation")
        if len(axes) != len(self.motion_bases):
            raise GridError("one base function identifier required per motion axis")
        for i, axis in enumerate(axes):
            _check_axis(axis, f"motion[{i}]")
        for name in self.motion_bases:
            if name not in MOTION_BASES:
                raise ConfigurationError(f"unknown base function {name!r}; known: {sorted(MOTION_BASES)}")
        elev.setflags(write=False)
        for axis in axes:
            axis.setflags(write=False)

    @property
    def shape(self) -> tuple:
        return (self.elevation.size,) + tuple(a.size for a in self.motion_axes)

    @property
    def flat_size(self) -> int:
        return int(np.prod(self.shape))

    @property
    def inner_size(self) -> int:
        """Number of flat columns per elevation bin (product of motion-axis sizes)."""
        return int(np.prod([a.size for a in self.motion_axes])) if self.motion_axes else 1

    def flat_to_multi(self, flat: int) -> tuple:
        if not 0 <= flat < self.flat_size:
            raise GridError(f"flat index {flat} out of range [0, {self.flat_size})")
        return tuple(int(i) for i in np.unravel_index(flat, self.shape))

    def values_at(self, flat: int) -> tuple:
        idx = self.flat_to_multi(flat)
        s = float(self.elevation[idx[0]])
        p = tuple(float(axis[i]) for axis, i in zip(self.motion_axes, idx[1:]))
        return s, p

    def elevation_profile(self, magnitudes: np.ndarray) -> np.ndarray:
        mags = np.asarray(magnitudes).reshape(self.shape)
        if mags.ndim == 1:
            return mags
        return mags.max(axis=tuple(range(1, mags.ndim)))

    @classmethod
    def uniform(cls, elevation_span, elevation_count: int, motion=()) -> "ParameterGrid":
        # model.py:217-235
        if elevation_count < 1:
            raise GridError("elevation_count must be >= 1")
        elev = np.linspace(elevation_span[0], elevation_span[1], elevation_count)
        axes, bases = [], []
        for base, lo, hi, count in motion:
            if count < 1:
                raise GridError("motion axis count must be >= 1")
            axes.append(np.linspace(lo, hi, count))
            bases.append(base)
        return cls(elevation=elev, motion_axes=tuple(axes), motion_bases=tuple(bases))
