"""Objective container and lambda rule mirrored from the reference ``prox.py``.

``Objective`` (prox.py:25-63) keeps the reference's validation and complex128 storage so the
single-pixel entry points accept exactly what the reference accepts; the arithmetic of every
proximal-gradient iteration (prox.py:66-150) runs fused inside the CUDA solver kernels.
``default_lambda`` (prox.py:153-161) runs on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import ConfigurationError

BACKTRACK_CAP = 50  # prox.py:22


@dataclass(frozen=True)
class Objective:
    """One L1LS instance: dictionary, measurement, regularization weight."""

    dictionary: np.ndarray
    measurement: np.ndarray
    lambda_reg: float

    def __post_init__(self):
        a = getattr(self.dictionary, "entries", self.dictionary)
        a = np.asarray(a, dtype=complex)
        b = np.asarray(self.measurement, dtype=complex).reshape(-1)
        object.__setattr__(self, "dictionary", a)
        object.__setattr__(self, "measurement", b)
        if a.ndim != 2:
            raise ConfigurationError("dictionary must be a 2-d matrix")
        if a.shape[0] != b.size:
            raise ConfigurationError(f"dictionary has {a.shape[0]} rows but measurement has {b.size} entries")
        if not (np.isfinite(self.lambda_reg) and self.lambda_reg >= 0):
            raise ConfigurationError(f"lambda_reg must be finite and >= 0, got {self.lambda_reg}")

    @property
    def shape(self) -> tuple:
        return self.dictionary.shape


def default_lambda(dictionary, measurement, beta: float = 0.05) -> float:
    """Scale-free default weight beta * ||A^H b||_inf, computed on the device (prox.py:153-161)."""
    from .solver import dictionary_for

    a = np.asarray(getattr(dictionary, "entries", dictionary))
    b = np.asarray(measurement).reshape(1, -1)
    if a.shape[1] == 0:
        return 0.0
    return float(dictionary_for(a).default_lambda(b, beta)[0].item())
