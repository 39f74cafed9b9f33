"""Multi-GPU plumbing: pixel sharding (cfg1-4) and column sharding of one huge dictionary (cfg5).

Pixel sharding: pixels are independent, so rank g solves its own contiguous
pixel range with no collective; the per-pixel seed rule depends only on the pixel id (cli.py:102),
so results are independent of the number of GPUs (the reference's worker-count invariance,
test_acceptance.py:266-312).

Column sharding (cfg5, m = 1,048,576): rank g owns a set of dictionary columns and the matching
slice of every iterate.  Each solver round runs the fused adjoint/prox/forward pass over the local
columns and produces the per-pixel partial forward product A_g z_g (n complex) plus three partial
sums; one all-reduce (NCCL over NVLink) makes them global, after which every rank applies the same
update.  For RBPG every reference block (solver.py:204-210) is striped across ranks, so block
identity -- and therefore the Lipschitz-weighted draw law -- is exactly the reference's.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .exceptions import ConfigurationError
from .solver import BatchSolution, Dictionary, SolverConfig, _torch, block_ranges


def pixel_shard(num_pixels: int, world: int, rank: int) -> tuple:
    """Contiguous pixel range [start, stop) of ``rank`` (sizes differ by at most one)."""
    base, rem = divmod(num_pixels, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def column_shards(m: int, world: int, num_blocks: int | None = None) -> list:
    """Per-rank lists of global column ranges, in local order.

    ``num_blocks`` None: one contiguous range per rank (ISTA/FISTA).  Otherwise every reference
    block b = [s_b, e_b) is split into ``world`` stripes and rank g owns stripe g of every block,
    so rank g's local block b is its g-th stripe of the global block b.
    """
    if world < 1:
        raise ConfigurationError("world size must be >= 1")
    if num_blocks is None:
        return [[pixel_shard(m, world, g)] for g in range(world)]
    out = [[] for _ in range(world)]
    for s, e in block_ranges(m, num_blocks):
        w = e - s
        if w < world:
            raise ConfigurationError(f"block of {w} columns cannot be striped over {world} ranks")
        for g in range(world):
            out[g].append((s + (g * w) // world, s + ((g + 1) * w) // world))
    return out


def local_columns(ranges) -> np.ndarray:
    """Global column indices of a rank's local columns (local order)."""
    return np.concatenate([np.arange(s, e) for s, e in ranges])


class ColumnShard:
    """One rank's slice of a column-sharded dictionary, with the GLOBAL Lipschitz constants."""

    def __init__(self, a_local, ranges, backend: str, num_blocks: int, lipschitz, device=None):
        self.ranges = list(ranges)
        self.backend = backend
        self.d = Dictionary(a_local, device=device)
        lib = self.d._lib
        if backend == "rbpg":
            j = len(self.ranges)
            if j != num_blocks:
                raise ConfigurationError("RBPG shard needs one stripe per block")
            widths = [e - s for s, e in self.ranges]
            starts = np.concatenate([[0], np.cumsum(widths)[:-1]]).astype(np.int64)
            stops = np.cumsum(widths).astype(np.int64)
            lip = np.asarray(lipschitz, dtype=float)
            _lib.check(lib.tb_set_partition(self.d.handle, j, (ctypes.c_int64 * j)(*starts), (ctypes.c_int64 * j)(*stops), (ctypes.c_double * j)(*lip)))
            self.d._active_j = num_blocks
            self.d._partitions[num_blocks] = None  # global partition set explicitly
        else:
            _lib.check(lib.tb_set_lipschitz(self.d.handle, float(lipschitz)))
            self.d._lip_full = float(lipschitz)


def solve_column_sharded(shards, pixels, lam, config: SolverConfig, seeds=None, reduce_fn=None, history: bool = False) -> list:
    """Drive the tiled solver round by round over one or several local shards.

    ``shards``: the ColumnShards this process owns (one per GPU rank in production; several on one
    device to emulate a multi-rank run).  ``reduce_fn(buffers)`` must sum the per-shard ``red``
    buffers in place across ALL shards of the job (e.g. torch.distributed.all_reduce for one local
    shard per rank); default: sum over the local shards.
    Returns one BatchSolution per local shard (x_hat holds that shard's local columns; objective,
    iterations and status are identical on every shard).
    """
    torch = _torch()
    backend = shards[0].backend
    p = int(pixels.shape[0])
    total = config.total_iters
    cfg = config.to_c()
    if reduce_fn is None:
        def reduce_fn(bufs):
            if len(bufs) > 1:
                s = bufs[0].clone()
                for b in bufs[1:]:
                    s += b.to(s.device)
                for b in bufs:
                    b.copy_(s.to(b.device))
    states = []
    for sh in shards:
        d = sh.d
        dev = d.device
        b = d._pixels(pixels)
        lam_t = torch.as_tensor(lam, dtype=torch.float64).reshape(-1).to(dev)
        seeds_t = None
        if backend == "rbpg":
            seeds_t = seeds.to(dev).view(torch.uint64) if isinstance(seeds, torch.Tensor) else torch.from_numpy(np.asarray(seeds, dtype=np.uint64)).to(dev)
        red = torch.zeros(p * (2 * d.n + 4), dtype=torch.float64, device=dev)
        hist = torch.full((p, total + 1), float("nan"), dtype=torch.float64, device=dev) if history else None
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _lib.check(d._lib.tb_tiled_create(d.handle, _lib.SOLVER_CODES[backend], ctypes.byref(cfg), _lib.ptr(b), _lib.ptr(lam_t), _lib.ptr(seeds_t), p,
                                               _lib.ptr(hist), total + 1 if history else 0, _lib.ptr(red), d._stream(), ctypes.byref(h)))
        states.append(dict(d=d, b=b, lam=lam_t, seeds=seeds_t, red=red, hist=hist, h=h))
    try:
        rem = ctypes.c_int64()
        for r in range(total * (cfg.backtrack_cap + 1) + 1):
            for s in states:
                with torch.cuda.device(s["d"].device):
                    _lib.check(s["d"]._lib.tb_tiled_round_a(s["h"], s["d"]._stream()))
            reduce_fn([s["red"] for s in states])
            for s in states:
                with torch.cuda.device(s["d"].device):
                    _lib.check(s["d"]._lib.tb_tiled_round_b(s["h"], s["d"]._stream()))
            if (r + 1) % 16 == 0 or r + 1 >= total:
                s = states[0]
                _lib.check(s["d"]._lib.tb_tiled_remaining(s["h"], ctypes.byref(rem), s["d"]._stream()))
                if rem.value == 0:
                    break
        out = []
        for s in states:
            d = s["d"]
            x = torch.empty((p, d.m), dtype=torch.complex64, device=d.device)
            ff = torch.empty(p, dtype=torch.float64, device=d.device)
            its = torch.empty(p, dtype=torch.int32, device=d.device)
            st = torch.empty(p, dtype=torch.int32, device=d.device)
            with torch.cuda.device(d.device):
                _lib.check(d._lib.tb_tiled_finish(s["h"], _lib.ptr(x), _lib.ptr(ff), _lib.ptr(its), _lib.ptr(st), d._stream()))
            res = BatchSolution(x_hat=x, objective_final=ff, iterations=its, status=st, history=s["hist"])
            res._no_append = backend != "rbpg"
            out.append(res)
        torch.cuda.synchronize()
        return out
    finally:
        for s in states:
            s["d"]._lib.tb_tiled_destroy(s["h"])


def gather_columns(local_x: list, shard_ranges: list, m: int):
    """Reassemble full x_hat [P, m] from per-shard local columns (host numpy)."""
    p = local_x[0].shape[0]
    full = np.zeros((p, m), dtype=np.complex64)
    for x, ranges in zip(local_x, shard_ranges):
        full[:, local_columns(ranges)] = np.asarray(x)
    return full
