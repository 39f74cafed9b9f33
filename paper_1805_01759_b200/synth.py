"""Seeded synthetic TomoSAR batches for the five BASELINE.json configurations.

The reference's paper data (TerraSAR-X stacks) is not available; these generators stand in
for it with the shapes, sizes and value distributions BASELINE.json states. They follow the
reference's pixel synthesis rule (``simulate.py:194-205``: g = sum_k a_k * steer_k + noise,
circular complex Gaussian noise with per-sample variance |a_ref|^2 10^(-SNR/10) taken from
the FIRST scatterer, ``simulate.py:77-83``) applied to the dictionary
A[i,k] = exp(-j 2 pi phase_i(k)) given in BASELINE.json.

Everything is host-side numpy input preparation (not the solve path): A and B are produced
in complex128 and rounded ONCE to complex64, which is what both the CUDA path and the fp64
oracle consume.  All randomness comes from numpy Philox substreams keyed
(config_seed, purpose, chunk) so the same config/seed always yields the same bytes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .grid import ParameterGrid

WAVELENGTH = 0.031  # metres; BASELINE cfg4/cfg5 phase uses 2*t*v/0.031 and 2*sin(2 pi t)*d/0.031

_CHUNK = 1 << 17


def _rng(seed: int, purpose: int, chunk: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed) & (2**64 - 1), (purpose << 32) | chunk]))


@dataclass
class SynthBatch:
    """One synthetic workload: shared dictionary, pixel stack, grid and truth."""

    name: str
    dictionary: np.ndarray  # complex64 [n, m] row-major (row = acquisition, col = flat grid index)
    pixels: np.ndarray  # complex64 [P, n]  (TSTK1 payload order, stack.py:46-52)
    grid: ParameterGrid
    k_max: int
    truth_support: list = field(default_factory=list)  # per pixel list of flat indices (small P only)
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.dictionary.shape[0])

    @property
    def m(self) -> int:
        return int(self.dictionary.shape[1])

    @property
    def num_pixels(self) -> int:
        return int(self.pixels.shape[0])


def elevation_dictionary(freqs: np.ndarray, elevations: np.ndarray) -> np.ndarray:
    """A[i,k] = exp(-j 2 pi f_i s_k) in complex128 (BASELINE.json cfg1-3)."""
    phase = np.outer(freqs, elevations)
    return np.exp(-2j * np.pi * phase)


def motion_dictionary(freqs, times, grid: ParameterGrid) -> np.ndarray:
    """A[i,k] = exp(-j 2 pi (f_i s + 2 t_i v / lambda + 2 sin(2 pi t_i) d / lambda)) (cfg4/cfg5).

    Flat index k enumerates the grid row-major with elevation leading (model.py:158-160).
    Velocity/seasonal axes are in metres (SURVEY.md section 8d unit decision).
    """
    s_ax, v_ax, d_ax = grid.elevation, grid.motion_axes[0], grid.motion_axes[1]
    n = freqs.size
    ps = np.outer(freqs, s_ax)  # [n, ns]
    pv = np.outer(2.0 * times / WAVELENGTH, v_ax)  # [n, nv]
    pd = np.outer(2.0 * np.sin(2.0 * np.pi * times) / WAVELENGTH, d_ax)  # [n, nd]
    phase = ps[:, :, None, None] + pv[:, None, :, None] + pd[:, None, None, :]
    return np.exp(-2j * np.pi * phase.reshape(n, -1))


def _pixels_from_truth(a128, positions, gains, sigma2, rng) -> np.ndarray:
    """b = sum_k gains[:,k] * A[:, positions[:,k]] + sqrt(sigma2/2)(N + jN), rounded to c64."""
    p, kmax = positions.shape
    n = a128.shape[0]
    b = np.zeros((p, n), dtype=np.complex128)
    for k in range(kmax):
        valid = positions[:, k] >= 0
        if not np.any(valid):
            continue
        cols = a128[:, positions[valid, k]].T  # [pv, n]
        b[valid] += gains[valid, k, None] * cols
    noise = rng.standard_normal((p, n)) + 1j * rng.standard_normal((p, n))
    b += np.sqrt(sigma2 / 2.0)[:, None] * noise
    return b.astype(np.complex64)


def _distinct_positions(rng, p: int, k: int, m: int) -> np.ndarray:
    pos = rng.integers(0, m, size=(p, k))
    if k >= 2:
        for _ in range(64):
            dup = np.zeros(p, dtype=bool)
            for a in range(k):
                for b in range(a + 1, k):
                    dup |= pos[:, a] == pos[:, b]
            if not dup.any():
                break
            pos[dup] = rng.integers(0, m, size=(int(dup.sum()), k))
    return pos


def make_config(cfg: int, num_pixels: int | None = None, seed: int = 2018) -> SynthBatch:
    """Build BASELINE.json configuration ``cfg`` (1..5); ``num_pixels`` truncates the batch.

    Pixel i of a truncated batch is identical to pixel i of the full batch (pixels are drawn
    in fixed chunks of 2^17 from per-chunk substreams).
    """
    if cfg not in (1, 2, 3, 4, 5):
        raise ValueError(f"unknown config {cfg}")
    geo = _rng(seed, 1, cfg)
    if cfg in (1, 2, 3):
        n, m, spacing, full_p = {1: (25, 200, 0.25, 1024), 2: (25, 300, 0.25, 1 << 20), 3: (50, 512, 0.125, 1 << 18)}[cfg]
        freqs = np.sort(geo.uniform(-0.5, 0.5, n))
        elev = (np.arange(m) - m // 2) * spacing
        grid = ParameterGrid(elevation=elev)
        a128 = elevation_dictionary(freqs, elev)
        k_max = 2
        meta = {"n": n, "m": m, "spacing": spacing, "freqs": freqs}
    elif cfg == 4:
        n, full_p = 100, 16384
        freqs = np.sort(geo.uniform(-0.5, 0.5, n))
        times = np.sort(geo.uniform(0.0, 4.0, n))
        elev = (np.arange(200) - 100) * 0.25
        grid = ParameterGrid(
            elevation=elev,
            motion_axes=(np.linspace(-0.02, 0.02, 40), np.linspace(0.0, 0.01, 20)),
            motion_bases=("linear", "seasonal"),
        )
        a128 = motion_dictionary(freqs, times, grid)
        m = a128.shape[1]
        k_max = 2
        meta = {"n": n, "m": m, "freqs": freqs, "times": times}
    else:
        n, full_p = 100, 64
        freqs = np.sort(geo.uniform(-0.5, 0.5, n))
        times = np.sort(geo.uniform(0.0, 4.0, n))
        elev = (np.arange(256) - 128) * 0.25
        grid = ParameterGrid(
            elevation=elev,
            motion_axes=(np.linspace(-0.02, 0.02, 64), np.linspace(0.0, 0.01, 64)),
            motion_bases=("linear", "seasonal"),
        )
        a128 = motion_dictionary(freqs, times, grid)
        m = a128.shape[1]
        k_max = 3
        meta = {"n": n, "m": m, "freqs": freqs, "times": times}

    p_total = full_p if num_pixels is None else int(num_pixels)
    if p_total > full_p:
        raise ValueError(f"config {cfg} has {full_p} pixels, asked for {p_total}")
    rayleigh = 1.0 / (freqs.max() - freqs.min())
    meta["rayleigh"] = rayleigh

    chunks = []
    supports = []
    for c0 in range(0, p_total, _CHUNK):
        pc = min(_CHUNK, p_total - c0)
        full_chunk = min(_CHUNK, full_p - c0)
        rng = _rng(seed, 2 + cfg, c0 // _CHUNK)
        if cfg == 1:
            kk = rng.choice(3, size=full_chunk, p=[0.2, 0.5, 0.3])
            pos = _distinct_positions(rng, full_chunk, 2, m)
            mag = rng.uniform(0.5, 1.5, (full_chunk, 2))
            ph = rng.uniform(0.0, 2 * np.pi, (full_chunk, 2))
            snr = np.full(full_chunk, 10.0)
            pos[kk < 2, 1] = -1
            pos[kk < 1, 0] = -1
            ref = np.where(kk > 0, mag[:, 0], 1.0)
        elif cfg == 2:
            kk = rng.integers(1, 3, size=full_chunk)
            kappa = rng.uniform(0.3, 1.5, full_chunk)
            sep = np.maximum(1, np.rint(kappa * rayleigh / spacing).astype(np.int64))
            first = rng.integers(0, m, size=full_chunk)
            lo = np.where(first + sep < m, first, first - sep)
            pos = np.stack([lo, lo + sep], axis=1)
            swap = rng.random(full_chunk) < 0.5
            pos[swap] = pos[swap][:, ::-1]
            mag = rng.uniform(0.5, 1.5, (full_chunk, 2))
            ph = rng.uniform(0.0, 2 * np.pi, (full_chunk, 2))
            snr = rng.uniform(0.0, 20.0, full_chunk)
            pos[kk < 2, 1] = -1
            ref = mag[:, 0]
        elif cfg == 3:
            kappa = rng.uniform(0.2, 0.8, full_chunk)
            sep = np.maximum(1, np.rint(kappa * rayleigh / spacing).astype(np.int64))
            first = rng.integers(0, m - sep)
            pos = np.stack([first, first + sep], axis=1)
            mag = np.ones((full_chunk, 2))
            ph = rng.uniform(0.0, 2 * np.pi, (full_chunk, 2))
            snr = np.full(full_chunk, 5.0)
            ref = mag[:, 0]
        elif cfg == 4:
            kk = rng.integers(1, 3, size=full_chunk)
            pos = _distinct_positions(rng, full_chunk, 2, m)
            mag = rng.uniform(0.5, 1.5, (full_chunk, 2))
            ph = rng.uniform(0.0, 2 * np.pi, (full_chunk, 2))
            snr = np.full(full_chunk, 10.0)
            pos[kk < 2, 1] = -1
            ref = mag[:, 0]
        else:
            pos = _distinct_positions(rng, full_chunk, 3, m)
            mag = rng.uniform(0.5, 1.5, (full_chunk, 3))
            ph = rng.uniform(0.0, 2 * np.pi, (full_chunk, 3))
            snr = np.full(full_chunk, 10.0)
            ref = mag[:, 0]
        gains = mag * np.exp(1j * ph)
        sigma2 = ref**2 * 10.0 ** (-snr / 10.0)
        chunks.append(_pixels_from_truth(a128, pos, gains, sigma2, _rng(seed, 16 + cfg, c0 // _CHUNK))[:pc])
        pos = pos[:pc]
        if p_total <= 65536:
            supports.extend([sorted(int(v) for v in row if v >= 0) for row in pos])
    pixels = np.concatenate(chunks, axis=0) if chunks else np.zeros((0, n), np.complex64)
    return SynthBatch(
        name=f"cfg{cfg}",
        dictionary=np.ascontiguousarray(a128.astype(np.complex64)),
        pixels=np.ascontiguousarray(pixels),
        grid=grid,
        k_max=k_max,
        truth_support=supports,
        meta=meta,
    )


def lambda_from_beta(dictionary: np.ndarray, pixels: np.ndarray, beta: float = 0.1) -> np.ndarray:
    """Host fp64 beta * max_k |(A^H b_p)_k| rounded to float32 (test/golden helper only)."""
    a = dictionary.astype(np.complex128)
    corr = pixels.astype(np.complex128) @ a.conj()
    return (beta * np.abs(corr).max(axis=1)).astype(np.float32)
