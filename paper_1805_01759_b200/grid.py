"""Parameter grid: the flat-index decode the selection stage needs.

Mirrors the reference ``ParameterGrid`` (``model.py:154-235``): the dictionary's flat column
index enumerates the grid row-major with elevation as the leading axis
(``model.py:158-160``), ``values_at`` decodes (elevation, motion coefficients)
(``model.py:203-208``) and ``elevation_profile`` collapses motion axes by max
(``model.py:210-215``).  ``build_steering_matrix`` builds the dense dictionary on the device
(``model.py:296-323``; SURVEY section 8f "next" row 2), whole or as one rank's column shard.
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


def build_steering_matrix(xi, grid: ParameterGrid, eta=None, sign: float = 1.0, col_range=None, device=None):
    """Dense steering dictionary on the device (model.py:296-323), complex64 torch tensor [n, m].

    ``xi``: spatial frequencies (n,) (model.py:254-259; BASELINE uses the normalised f_i with
    sign=-1); ``eta``: temporal frequencies (n_axes, n) (model.py:262-277), one row per motion axis.
    ``col_range`` (start, stop) builds one column shard only.  No 50M-entry budget: the dictionary
    lives in HBM (cfg5's 100 x 1,048,576 = 800 MiB).
    """
    import ctypes

    import torch

    from . import _lib
    from .exceptions import NumericalError

    if not torch.cuda.is_available():
        raise NumericalError("no CUDA device: the B200 solver has no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
    xi_t = torch.as_tensor(np.asarray(xi, dtype=np.float64)).to(dev)
    n = int(xi_t.numel())
    n_axes = len(grid.motion_axes)
    eta_np = np.zeros((max(n_axes, 1), n)) if eta is None else np.asarray(eta, dtype=np.float64).reshape(n_axes, n)
    eta_t = torch.as_tensor(np.ascontiguousarray(eta_np)).to(dev)
    elev_t = torch.as_tensor(np.array(grid.elevation, dtype=np.float64)).to(dev)
    mot = np.concatenate([np.asarray(a, dtype=np.float64) for a in grid.motion_axes]) if n_axes else np.zeros(1)
    mot_t = torch.as_tensor(mot).to(dev)
    sizes = (ctypes.c_int32 * max(1, n_axes))(*([a.size for a in grid.motion_axes] or [1]))
    c0, c1 = (0, grid.flat_size) if col_range is None else (int(col_range[0]), int(col_range[1]))
    out = torch.empty((n, c1 - c0), dtype=torch.complex64, device=dev)
    lib = _lib.load()
    with torch.cuda.device(dev):
        _lib.check(lib.tb_build_steering(dev.index, _lib.ptr(xi_t), _lib.ptr(eta_t), n, n_axes, _lib.ptr(elev_t), int(grid.elevation.size),
                                         _lib.ptr(mot_t), sizes, c0, c1 - c0, float(sign), _lib.ptr(out), torch.cuda.current_stream(dev).cuda_stream))
    return out
