"""Solver entry points mirroring the reference ``solver.py``, executed by the sm_100a library.

Drop-in names and layouts (reference file:line, relative to /root/reference/pkg/src/tomobpdn):
``SolverConfig`` (solver.py:35-97), ``config_schema`` (:100-116), ``SolverStatus`` (:119-123),
``Solution`` (:126-134), ``BlockPartition`` (:137-164), ``spectral_sq_norm`` (:167-188),
``block_partition`` (:191-214), ``rbpg_solve`` (:250-338), ``ista_solve`` (:379-381),
``fista_solve`` (:384-390).  The batch entry ``Dictionary.solve`` runs one fused persistent
kernel over a whole pixel stack; the single-pixel functions wrap a batch of one.

Compute happens only in ``lib/libtomobpdn_b200.so``; torch is used for device buffers and
streams.  There is no CPU fallback: without the library or a GPU these functions raise.
"""

from __future__ import annotations

import ctypes
import os
import hashlib
import json
import time
from collections import OrderedDict
from dataclasses import dataclass, field, fields
from enum import Enum
from pathlib import Path

import numpy as np

from . import _lib
from .exceptions import ConfigurationError, NumericalError

STOP_WINDOW = 10  # solver.py:29
THETA_SCHEDULE = "2/(k+1)"  # solver.py:30
BACKTRACK_CAP = 50  # prox.py:22
_POWER_ITER_SEED = 0x5EED0F  # solver.py:32


@dataclass(frozen=True)
class SolverConfig:
    """Tuning knobs shared by all iterative solvers (same fields, defaults, validation)."""

    lambda_reg: float | None = None
    num_blocks: int = 8
    max_iters: int = 5000
    tol: float = 1e-8
    c_alpha: float = 0.5
    alpha_init_scale: float = 1.0
    seed: int = 0
    fixed_iters: int | None = None
    theta_schedule: str = THETA_SCHEDULE

    def __post_init__(self):
        if self.lambda_reg is not None and not (np.isfinite(self.lambda_reg) and self.lambda_reg >= 0):
            raise ConfigurationError(f"lambda_reg must be >= 0, got {self.lambda_reg}")
        if self.num_blocks < 1:
            raise ConfigurationError(f"num_blocks must be >= 1, got {self.num_blocks}")
        if self.max_iters < 1:
            raise ConfigurationError(f"max_iters must be >= 1, got {self.max_iters}")
        if not (np.isfinite(self.tol) and self.tol > 0):
            raise ConfigurationError(f"tol must be > 0, got {self.tol}")
        if not 0.0 < self.c_alpha < 1.0:
            raise ConfigurationError(f"c_alpha must lie in (0, 1), got {self.c_alpha}")
        if not (np.isfinite(self.alpha_init_scale) and self.alpha_init_scale > 0):
            raise ConfigurationError(f"alpha_init_scale must be > 0, got {self.alpha_init_scale}")
        if self.fixed_iters is not None and self.fixed_iters < 1:
            raise ConfigurationError(f"fixed_iters must be >= 1, got {self.fixed_iters}")
        if self.theta_schedule != THETA_SCHEDULE:
            raise ConfigurationError(f"theta_schedule is pinned to {THETA_SCHEDULE!r}, got {self.theta_schedule!r}")

    def to_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @classmethod
    def from_dict(cls, data: dict) -> "SolverConfig":
        known = {f.name for f in fields(cls)}
        unknown = set(data) - known
        if unknown:
            raise ConfigurationError(f"unknown solver config keys: {sorted(unknown)}")
        return cls(**data)

    @classmethod
    def from_json(cls, path) -> "SolverConfig":
        with open(path, "r", encoding="utf-8") as fh:
            return cls.from_dict(json.load(fh))

    def to_c(self) -> _lib.SolverConfigC:
        return _lib.SolverConfigC(
            num_blocks=int(self.num_blocks),
            max_iters=int(self.max_iters),
            fixed_iters=int(self.fixed_iters or 0),
            backtrack_cap=BACKTRACK_CAP,
            tol=float(self.tol),
            c_alpha=float(self.c_alpha),
            alpha_init_scale=float(self.alpha_init_scale),
        )

    @property
    def total_iters(self) -> int:
        return int(self.fixed_iters if self.fixed_iters is not None else self.max_iters)


def config_schema() -> dict:
    """Machine-readable description of all solver knobs and their defaults (solver.py:100-116)."""
    type_names = {
        "lambda_reg": "float | null",
        "num_blocks": "int",
        "max_iters": "int",
        "tol": "float",
        "c_alpha": "float",
        "alpha_init_scale": "float",
        "seed": "int",
        "fixed_iters": "int | null",
        "theta_schedule": "str (pinned)",
    }
    return {f.name: {"type": type_names[f.name], "default": f.default} for f in fields(SolverConfig)}


class SolverStatus(str, Enum):
    CONVERGED = "converged"
    MAX_ITERS = "max-iters"
    LINE_SEARCH_FAILURE = "line-search-failure"
    NUMERICAL_FAILURE = "numerical-failure"


STATUS_BY_CODE = (SolverStatus.CONVERGED, SolverStatus.MAX_ITERS, SolverStatus.LINE_SEARCH_FAILURE, SolverStatus.NUMERICAL_FAILURE)


@dataclass(frozen=True)
class Solution:
    """Recovered reflectivity vector plus convergence telemetry."""

    x_hat: np.ndarray
    objective_history: np.ndarray
    iterations_used: int
    status: SolverStatus
    wall_time: float


@dataclass(frozen=True)
class BlockPartition:
    """Contiguous coordinate blocks with Lipschitz-weighted sampling law (solver.py:137-164)."""

    blocks: tuple
    lipschitz: np.ndarray
    probabilities: np.ndarray = field(init=False)

    def __post_init__(self):
        lip = np.asarray(self.lipschitz, dtype=float)
        if lip.size != len(self.blocks):
            raise ConfigurationError("one Lipschitz constant required per block")
        if np.any(lip < 0) or not np.all(np.isfinite(lip)):
            raise ConfigurationError("Lipschitz constants must be finite and >= 0")
        stop_prev = self.blocks[0][0]
        for start, stop in self.blocks:
            if start != stop_prev or stop <= start:
                raise ConfigurationError("blocks must be contiguous, disjoint, non-empty")
            stop_prev = stop
        total = float(lip.sum())
        if total <= 0:
            raise ConfigurationError("at least one block must have positive Lipschitz")
        object.__setattr__(self, "lipschitz", lip)
        object.__setattr__(self, "probabilities", lip / total)

    @property
    def num_blocks(self) -> int:
        return len(self.blocks)


def block_ranges(l_total: int, num_blocks: int) -> tuple:
    """Near-equal contiguous blocks, the first l_total mod J one longer (solver.py:204-210)."""
    if not 1 <= num_blocks <= l_total:
        raise ConfigurationError(f"num_blocks must lie in [1, {l_total}], got {num_blocks}")
    base, rem = divmod(l_total, num_blocks)
    out, start = [], 0
    for i in range(num_blocks):
        stop = start + base + (1 if i < rem else 0)
        out.append((start, stop))
        start = stop
    return tuple(out)


def _power_start_vector(n_cols: int) -> np.ndarray:
    # substream(0x5EED0F, n_cols) normals, normalised (solver.py:171-173); host input prep
    g = np.random.Generator(np.random.Philox(key=[_POWER_ITER_SEED, n_cols]))
    v = g.standard_normal(n_cols) + 1j * g.standard_normal(n_cols)
    return v / np.linalg.norm(v)


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise NumericalError("no CUDA device: the B200 solver has no CPU fallback")
    return torch


@dataclass
class BatchSolution:
    """Per-pixel solver outputs of one batch (device tensors)."""

    x_hat: object  # complex64 [P, m]
    objective_final: object  # float64 [P]
    iterations: object  # int32 [P]
    status: object  # int32 [P]
    history: object = None  # float64 [P, T+1] (NaN padded) or None
    wall_time: float = 0.0

    def solution(self, i: int) -> Solution:
        it = int(self.iterations[i].item())
        st = STATUS_BY_CODE[int(self.status[i].item())]
        if self.history is not None:
            n_hist = it if (st == SolverStatus.LINE_SEARCH_FAILURE and self._no_append) else it + 1
            hist = self.history[i, :n_hist].cpu().numpy()
        else:
            hist = np.array([float(self.objective_final[i].item())])
        x = self.x_hat[i].cpu().numpy().astype(np.complex128)
        return Solution(x_hat=x, objective_history=hist, iterations_used=it, status=st, wall_time=self.wall_time)

    _no_append: bool = False


class Dictionary:
    """A steering dictionary resident on one GPU plus its per-dictionary setup.

    Wraps a ``tb_ctx``.  The Lipschitz constants (whole matrix for ISTA/FISTA, per block for
    RBPG) are computed once per dictionary on the device (the reference recomputes them in
    every solve, solver.py:267, 344) and cached.
    """

    def __init__(self, a, device=None):
        torch = _torch()
        lib = _lib.load()
        if device is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        elif isinstance(device, torch.device):
            dev = device if device.index is not None else torch.device("cuda", torch.cuda.current_device())
        else:
            dev = torch.device("cuda", int(device))
        if isinstance(a, torch.Tensor):
            at = a.to(device=dev, dtype=torch.complex64).contiguous()
        else:
            arr = np.asarray(a)
            if arr.ndim != 2:
                raise ConfigurationError("dictionary must be a 2-d matrix")
            at = torch.from_numpy(np.ascontiguousarray(arr.astype(np.complex64))).to(dev)
        if at.ndim != 2:
            raise ConfigurationError("dictionary must be a 2-d matrix")
        self.device = dev
        self.n, self.m = int(at.shape[0]), int(at.shape[1])
        self.tensor = at
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _lib.check(lib.tb_ctx_create(dev.index, _lib.ptr(at), self.n, self.m, ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self._pid = os.getpid()  # a forked child (e.g. a CPU process pool) must not touch the context
        self._lip_full = None
        self._partitions = {}
        self._active_j = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and getattr(self, "_pid", None) == os.getpid():
            try:
                self._lib.tb_ctx_destroy(h)
            except Exception:
                pass

    @property
    def handle(self):
        return self._h

    def _stream(self):
        torch = _torch()
        return torch.cuda.current_stream(self.device).cuda_stream

    def spectral_sq_norms(self, ranges, max_iter: int = 300, rtol: float = 1e-12) -> np.ndarray:
        """sigma_max^2 of each column range by fp64 device power iteration (solver.py:167-188)."""
        torch = _torch()
        starts = (ctypes.c_int64 * len(ranges))(*[int(s) for s, _ in ranges])
        stops = (ctypes.c_int64 * len(ranges))(*[int(e) for _, e in ranges])
        v0 = np.concatenate([_power_start_vector(int(e - s)) if e - s > 1 else np.ones(1, complex) for s, e in ranges])
        v0t = torch.from_numpy(v0.astype(np.complex128)).to(self.device)
        out = (ctypes.c_double * len(ranges))()
        with torch.cuda.device(self.device):
            _lib.check(self._lib.tb_spectral_sq_norms(self._h, len(ranges), starts, stops, _lib.ptr(v0t), max_iter, rtol, out, self._stream()))
        return np.array(list(out), dtype=float)

    def lipschitz(self) -> float:
        """L = 2 sigma_max(A)^2 (solver.py:344)."""
        if self._lip_full is None:
            self._lip_full = 2.0 * float(self.spectral_sq_norms([(0, self.m)])[0])
            _lib.check(self._lib.tb_set_lipschitz(self._h, self._lip_full))
        return self._lip_full

    def partition(self, num_blocks: int) -> BlockPartition:
        """block_partition (solver.py:191-214) computed once per (dictionary, J)."""
        if num_blocks not in self._partitions:
            ranges = block_ranges(self.m, num_blocks)
            lip = 2.0 * self.spectral_sq_norms(ranges)
            self._partitions[num_blocks] = BlockPartition(blocks=ranges, lipschitz=lip)
        part = self._partitions[num_blocks]
        if self._active_j != num_blocks:
            j = part.num_blocks
            starts = (ctypes.c_int64 * j)(*[s for s, _ in part.blocks])
            stops = (ctypes.c_int64 * j)(*[e for _, e in part.blocks])
            lips = (ctypes.c_double * j)(*[float(v) for v in part.lipschitz])
            _lib.check(self._lib.tb_set_partition(self._h, j, starts, stops, lips))
            self._active_j = num_blocks
        return part

    def _pixels(self, pixels):
        torch = _torch()
        if isinstance(pixels, torch.Tensor):
            t = pixels.to(device=self.device, dtype=torch.complex64)
        else:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(pixels).astype(np.complex64))).to(self.device)
        if t.ndim == 1:
            t = t.reshape(1, -1)
        if t.ndim != 2 or t.shape[1] != self.n:
            raise ConfigurationError(f"dictionary has {self.n} rows but measurements have shape {tuple(t.shape)}")
        return t.contiguous()

    def default_lambda(self, pixels, beta: float = 0.05):
        """beta * max |A^H b| per pixel, float64 device tensor (prox.py:153-161)."""
        torch = _torch()
        b = self._pixels(pixels)
        lam = torch.empty(b.shape[0], dtype=torch.float64, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(self._lib.tb_default_lambda(self._h, _lib.ptr(b), b.shape[0], float(beta), _lib.ptr(lam), self._stream()))
        return lam

    def derive_seeds(self, run_seed: int, num_pixels: int, first_pixel_id: int = 0):
        """derive_seed(substream(run_seed, pixel_id)) per pixel on device (cli.py:102)."""
        torch = _torch()
        seeds = torch.empty(num_pixels, dtype=torch.uint64, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(self._lib.tb_derive_seeds(int(run_seed) & (2**64 - 1), int(first_pixel_id), int(num_pixels), _lib.ptr(seeds), self._stream()))
        return seeds

    def synthesize_pairs(self, seed: int, stream_ids, col0, col1, phase, sigma):
        """Two-scatterer Monte-Carlo realizations on the device (tb_synthesize_pairs; simulate.py:297-335):
        pixels[r] = A[:, col0[r]] + e^{j phase[r]} A[:, col1[r]] + complex normal noise of variance sigma[r]^2
        (phase NaN = drawn), plus each realization's nested RBPG seed.  Statistically equivalent to
        the reference's draws (Philox substreams, Box-Muller normals).  Returns (pixels c64 [R, n],
        seeds u64 [R]) on this device."""
        torch = _torch()
        dev = self.device
        sid = torch.as_tensor(np.asarray(stream_ids, dtype=np.uint64).astype(np.int64)).to(dev).view(torch.uint64)
        c0 = torch.as_tensor(np.asarray(col0, dtype=np.int32)).to(dev)
        c1 = torch.as_tensor(np.asarray(col1, dtype=np.int32)).to(dev)
        ph = torch.as_tensor(np.asarray(phase, dtype=np.float32)).to(dev)
        sg = torch.as_tensor(np.asarray(sigma, dtype=np.float32)).to(dev)
        r = int(sid.numel())
        if not (c0.numel() == c1.numel() == ph.numel() == sg.numel() == r):
            raise ConfigurationError("one column pair, phase and sigma per realization")
        if r and (int(min(c0.min(), c1.min())) < 0 or int(max(c0.max(), c1.max())) >= self.m):
            raise ConfigurationError("scatterer columns outside the dictionary")
        pix = torch.empty((r, self.n), dtype=torch.complex64, device=dev)
        seeds = torch.empty(r, dtype=torch.uint64, device=dev)
        with torch.cuda.device(dev):
            _lib.check(self._lib.tb_synthesize_pairs(self._h, int(seed) & (2**64 - 1), _lib.ptr(sid), _lib.ptr(c0), _lib.ptr(c1),
                                                     _lib.ptr(ph), _lib.ptr(sg), r, _lib.ptr(pix), _lib.ptr(seeds), self._stream()))
        return pix, seeds

    def solve(self, pixels, lam, config: SolverConfig, backend: str = "rbpg", seeds=None, history: bool = False, out=None, path: str = "auto", allreduce=None) -> BatchSolution:
        """Solve every pixel of a stack on the device.

        ``path`` "auto" lets the library pick the warp-per-pixel kernel (dictionary and iterate in
        shared memory) or the tiled large-dictionary solver; "tiled" forces the latter, driven
        round by round from here so that ``allreduce(red)`` (sum over column shards, e.g.
        torch.distributed.all_reduce) can run between the pass and the update.
        """
        torch = _torch()
        if backend not in _lib.SOLVER_CODES:
            raise ConfigurationError(f"unknown iterative backend {backend!r}")
        b = self._pixels(pixels)
        p = int(b.shape[0])
        if not isinstance(lam, torch.Tensor):
            lam_h = np.asarray(lam, dtype=np.float64).reshape(-1)
            if not (np.all(np.isfinite(lam_h)) and np.all(lam_h >= 0)):
                raise ConfigurationError("lambda_reg must be finite and >= 0")  # prox.py:47-48
        lam_t = torch.as_tensor(lam, dtype=torch.float64).reshape(-1).to(self.device)
        if lam_t.numel() == 1 and p != 1:
            lam_t = lam_t.expand(p).contiguous()
        if lam_t.numel() != p:
            raise ConfigurationError(f"need one lambda per pixel ({p}), got {lam_t.numel()}")
        seeds_t = None
        if backend == "rbpg":
            self.partition(config.num_blocks)
            if seeds is None:
                seeds = np.full(p, int(config.seed) & (2**64 - 1), dtype=np.uint64)
            if isinstance(seeds, torch.Tensor):
                if seeds.dtype not in (torch.int64, torch.uint64):
                    raise ConfigurationError("seeds must be an int64/uint64 tensor")
                seeds_t = seeds.to(self.device).contiguous().view(torch.uint64)
            else:
                seeds_t = torch.from_numpy(np.asarray(seeds, dtype=np.uint64).reshape(-1)).to(self.device)
            if seeds_t.numel() != p:
                raise ConfigurationError("need one seed per pixel")
        else:
            self.lipschitz()
        total = config.total_iters
        if out is None:
            x = torch.empty((p, self.m), dtype=torch.complex64, device=self.device)
            ffin = torch.empty(p, dtype=torch.float64, device=self.device)
            its = torch.empty(p, dtype=torch.int32, device=self.device)
            st = torch.empty(p, dtype=torch.int32, device=self.device)
        else:
            x, ffin, its, st = out
        hist = torch.full((p, total + 1), float("nan"), dtype=torch.float64, device=self.device) if history else None
        cfg = config.to_c()
        t0 = time.perf_counter()
        if path == "tiled" or allreduce is not None:
            self._solve_tiled(backend, cfg, b, lam_t, seeds_t, p, x, ffin, hist, total, its, st, allreduce)
            res = BatchSolution(x_hat=x, objective_final=ffin, iterations=its, status=st, history=hist, wall_time=time.perf_counter() - t0)
            res._no_append = backend != "rbpg"
            return res
        with torch.cuda.device(self.device):
            _lib.check(
                self._lib.tb_solve(
                    self._h, _lib.SOLVER_CODES[backend], ctypes.byref(cfg), _lib.ptr(b), _lib.ptr(lam_t), _lib.ptr(seeds_t), p,
                    _lib.ptr(x), _lib.ptr(ffin), _lib.ptr(hist), total + 1 if history else 0, _lib.ptr(its), _lib.ptr(st), self._stream(),
                )
            )
        res = BatchSolution(x_hat=x, objective_final=ffin, iterations=its, status=st, history=hist, wall_time=time.perf_counter() - t0)
        res._no_append = backend != "rbpg"
        return res


    def wiener_filter(self, noise_power: float):
        """W = V diag(s / (s^2 + mu)) U^H from the thin SVD of A (solver.py:393-407), cached per mu.

        The SVD (cuSOLVER, complex128, n x m with n <= 128) is a once-per-dictionary setup step on
        the device; applying W to the pixel stack is the batched kernel ``tb_apply_filter``.
        """
        torch = _torch()
        if not (np.isfinite(noise_power) and noise_power >= 0):
            raise ConfigurationError(f"noise_power must be >= 0, got {noise_power}")
        cache = self.__dict__.setdefault("_wiener", {})
        if noise_power not in cache:
            try:
                u, s, vh = torch.linalg.svd(self.tensor.to(torch.complex128), full_matrices=False)
            except RuntimeError as exc:
                raise NumericalError(f"SVD failed: {exc}") from exc
            filt = s / (s * s + noise_power)
            cache[noise_power] = (vh.conj().transpose(0, 1) * filt.to(torch.complex128)[None, :]) @ u.conj().transpose(0, 1)
            cache[noise_power] = cache[noise_power].contiguous()
        return cache[noise_power]

    def wiener(self, pixels, noise_power: float):
        """svd_wiener_solve for every pixel: complex64 x_hat [P, m] (solver.py:393-407)."""
        torch = _torch()
        w = self.wiener_filter(noise_power)
        b = self._pixels(pixels)
        x = torch.empty((b.shape[0], self.m), dtype=torch.complex64, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(self._lib.tb_apply_filter(self._h, _lib.ptr(w), _lib.ptr(b), b.shape[0], _lib.ptr(x), self._stream()))
        return x

    def _solve_tiled(self, backend, cfg, b, lam_t, seeds_t, p, x, ffin, hist, total, its, st, allreduce):
        torch = _torch()
        if p == 0:
            return
        red = torch.zeros(p * (2 * self.n + 4), dtype=torch.float64, device=self.device)
        h = ctypes.c_void_p()
        stream = self._stream()
        with torch.cuda.device(self.device):
            _lib.check(
                self._lib.tb_tiled_create(
                    self._h, _lib.SOLVER_CODES[backend], ctypes.byref(cfg), _lib.ptr(b), _lib.ptr(lam_t), _lib.ptr(seeds_t), p,
                    _lib.ptr(hist), total + 1 if hist is not None else 0, _lib.ptr(red), stream, ctypes.byref(h),
                )
            )
            try:
                rem = ctypes.c_int64()
                max_rounds = total * (cfg.backtrack_cap + 1) + 1
                for r in range(max_rounds):
                    _lib.check(self._lib.tb_tiled_round_a(h, stream))
                    if allreduce is not None:
                        allreduce(red)
                    _lib.check(self._lib.tb_tiled_round_b(h, stream))
                    if (r + 1) % 16 == 0 or r + 1 >= total:
                        _lib.check(self._lib.tb_tiled_remaining(h, ctypes.byref(rem), stream))
                        if rem.value == 0:
                            break
                _lib.check(self._lib.tb_tiled_finish(h, _lib.ptr(x), _lib.ptr(ffin), _lib.ptr(its), _lib.ptr(st), stream))
                torch.cuda.synchronize(self.device)
            finally:
                self._lib.tb_tiled_destroy(h)


_CACHE: "OrderedDict[tuple, Dictionary]" = OrderedDict()


def dictionary_for(a, device=None) -> Dictionary:
    """Context cache keyed by dictionary content, so repeated per-pixel calls reuse setup."""
    if isinstance(a, Dictionary):
        return a
    arr = np.asarray(getattr(a, "entries", a))
    key = (arr.shape, hashlib.sha1(np.ascontiguousarray(arr.astype(np.complex64)).view(np.uint8)).hexdigest(), device)
    d = _CACHE.get(key)
    if d is None:
        d = Dictionary(arr, device=device)
        _CACHE[key] = d
        while len(_CACHE) > 8:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    return d


def spectral_sq_norm(a, max_iter: int = 300, rtol: float = 1e-12) -> float:
    """Largest squared singular value by device power iteration (solver.py:167-188)."""
    d = dictionary_for(a)
    return float(d.spectral_sq_norms([(0, d.m)], max_iter, rtol)[0])


def block_partition(l_total: int, num_blocks: int, a) -> BlockPartition:
    """Contiguous blocks with per-block Lipschitz 2 sigma_max(A_i)^2 (solver.py:191-214)."""
    arr = np.asarray(getattr(a, "entries", a))
    if not 1 <= num_blocks <= l_total:
        raise ConfigurationError(f"num_blocks must lie in [1, {l_total}], got {num_blocks}")
    if arr.shape[1] != l_total:
        raise ConfigurationError("matrix column count must equal l_total")
    return dictionary_for(arr).partition(num_blocks)


def _single(obj, config: SolverConfig, backend: str) -> Solution:
    from .prox import Objective

    if not isinstance(obj, Objective):
        raise ConfigurationError("expected an Objective")
    t0 = time.perf_counter()
    d = dictionary_for(obj.dictionary)
    if backend == "rbpg" and not 1 <= config.num_blocks <= d.m:
        raise ConfigurationError(f"num_blocks must lie in [1, {d.m}], got {config.num_blocks}")
    seeds = np.array([int(config.seed) & (2**64 - 1)], dtype=np.uint64) if backend == "rbpg" else None
    bs = d.solve(obj.measurement.reshape(1, -1), np.array([obj.lambda_reg]), config, backend, seeds=seeds, history=True)
    sol = bs.solution(0)
    return Solution(sol.x_hat, sol.objective_history, sol.iterations_used, sol.status, time.perf_counter() - t0)


def rbpg_solve(obj, config: SolverConfig) -> Solution:
    """Randomized blockwise proximal gradient with backtracking (solver.py:250-338)."""
    return _single(obj, config, "rbpg")


def ista_solve(obj, config: SolverConfig) -> Solution:
    """Plain proximal gradient with backtracking (solver.py:379-381)."""
    return _single(obj, config, "ista")


def fista_solve(obj, config: SolverConfig) -> Solution:
    """Nesterov-accelerated full-vector proximal gradient (solver.py:384-390)."""
    return _single(obj, config, "fista")


def sample_block(partition: BlockPartition, rng) -> int:
    """Lipschitz-weighted block draw with numpy's choice rule (solver.py:217-219).

    Host helper kept for API parity; the solver kernels draw in-kernel with Philox4x64-10.
    """
    return int(rng.choice(partition.num_blocks, p=partition.probabilities))


def svd_wiener_solve(obj, noise_power: float) -> np.ndarray:
    """Wiener/Tikhonov-regularised pseudo-inverse profile V diag(s/(s^2+mu)) U^H g (solver.py:393-407)."""
    from .prox import Objective

    if not isinstance(obj, Objective):
        raise ConfigurationError("expected an Objective")
    d = dictionary_for(obj.dictionary)
    return d.wiener(obj.measurement.reshape(1, -1), noise_power)[0].cpu().numpy().astype(np.complex128)
