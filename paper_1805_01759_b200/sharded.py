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


# ------------------------------------------------------------------ pixel-sharded pipeline (cfg1-4)

_EST_FIELDS = ("model_order", "support", "amplitudes", "elevations", "motion_params", "selection_scores", "n_scores", "error")
_SOL_FIELDS = ("objective_final", "iterations", "status")


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def _all_gather_rows(t, spans, group):
    """Ordered all-gather of a per-rank row block (contiguous pixel shards, sizes differ by <= 1).
    Host plumbing: works on CPU tensors too (gloo), so it is tested without a GPU."""
    import torch

    dist = _dist()
    rows = max(e - s for s, e in spans)
    real = torch.view_as_real(t) if t.is_complex() else t
    home = real.device
    if dist.get_backend(group) == "gloo":  # gloo gathers host tensors; NCCL gathers in HBM
        real = real.cpu()
    pad = torch.zeros((rows,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
    pad[: real.shape[0]] = real
    bufs = [torch.empty_like(pad) for _ in spans]
    dist.all_gather(bufs, pad, group=group)
    out = torch.cat([b[: e - s] for b, (s, e) in zip(bufs, spans)]).to(home)
    return torch.view_as_complex(out) if t.is_complex() else out


def gather_estimates(est, num_pixels: int, group=None):
    """All ranks' contiguous-shard ``BatchEstimates`` -> the whole batch's, in pixel order, on every
    rank (one all-gather per field over the job's process group: NCCL on GPUs).  The pixel order of
    the output equals the input order for any world size, as the reference's ordered ``pool.map``
    output (cli.py:136-144)."""
    from .slimmer import BatchEstimates

    dist = _dist()
    world = dist.get_world_size(group)
    spans = [pixel_shard(num_pixels, world, g) for g in range(world)]
    fields = {f: _all_gather_rows(getattr(est, f), spans, group) for f in _EST_FIELDS}
    out = BatchEstimates(**fields)
    if est.solution is not None:
        sol = {f: _all_gather_rows(getattr(est.solution, f), spans, group) for f in _SOL_FIELDS}
        x = _all_gather_rows(est.solution.x_hat, spans, group) if est.solution.x_hat is not None else None
        out.solution = BatchSolution(x_hat=x, history=None, wall_time=est.solution.wall_time, **sol)
        out.solution._no_append = getattr(est.solution, "_no_append", False)
    if est.lam is not None and hasattr(est.lam, "is_complex"):
        out.lam = _all_gather_rows(est.lam, spans, group)
    return out


def pipeline_sharded(dictionary, pixels, grid, config, beta: float = 0.05, run_seed=None, devices=None, group=None,
                     gather: bool = True, keep_x: bool = True):
    """The batched pipeline with the pixel batch sharded over GPUs.

    Pixels are independent, so every GPU solves a contiguous pixel range with NO collective on the
    data path; per-pixel seeds depend only on the global pixel id (cli.py:102), so every output is
    bit-identical for any number of GPUs (the reference's worker-count invariance,
    test_acceptance.py:266-312).

    * ``torch.distributed`` initialised (one process per GPU, e.g. torchrun): this rank takes
      ``pixel_shard(P, world, rank)`` of ``pixels`` (the whole batch, on the host or any device) and,
      with ``gather``, the ranks all-gather the estimates in pixel order (the output collection).
    * otherwise ``devices`` (a list of CUDA devices) shards the batch inside one process: the
      shards' work is enqueued on every device before any result is collected, so the GPUs run
      concurrently; results are concatenated on ``devices[0]``.
    ``dictionary``: the matrix, or a Dictionary per device (a dict device -> Dictionary) to reuse
    contexts.  Returns BatchEstimates for the whole batch (or, ``gather=False``, this rank's shard).
    """
    from .slimmer import BatchEstimates, pipeline_batch

    torch = _torch()
    p = int(pixels.shape[0])
    seed = config.solver.seed if run_seed is None else run_seed
    dist = _dist()

    def norm(dev):
        if dev is None:
            return torch.device("cuda", torch.cuda.current_device())
        return dev if isinstance(dev, torch.device) else torch.device("cuda", int(dev))

    def ctx(dev):
        dev = norm(dev)
        if isinstance(dictionary, dict):
            return dictionary[dev.index] if dev.index in dictionary else dictionary[dev]
        if isinstance(dictionary, Dictionary):
            if dev != dictionary.device:
                raise ConfigurationError("a single Dictionary can only serve its own device")
            return dictionary
        return Dictionary(dictionary, device=dev)

    def shard(rows):
        s, e = rows
        return pixels[s:e]

    if dist is not None:
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        s, e = pixel_shard(p, world, rank)
        est = pipeline_batch(ctx(None), shard((s, e)), grid, config, beta=beta, run_seed=seed, first_pixel_id=s)
        if not keep_x:
            est.solution.x_hat = None
        return gather_estimates(est, p, group) if gather else est
    devs = [norm(x) for x in (devices or [None])]
    spans = [pixel_shard(p, len(devs), g) for g in range(len(devs))]
    parts = []
    for dev, (s, e) in zip(devs, spans):  # enqueue every shard before touching any result
        with torch.cuda.device(dev):
            parts.append(pipeline_batch(ctx(dev), shard((s, e)), grid, config, beta=beta, run_seed=seed, first_pixel_id=s))
    home = devs[0]
    cat = lambda ts: torch.cat([t.to(home) for t in ts])  # noqa: E731
    out = BatchEstimates(**{f: cat([getattr(q, f) for q in parts]) for f in _EST_FIELDS})
    sols = [q.solution for q in parts]
    out.solution = BatchSolution(x_hat=cat([q.x_hat for q in sols]) if keep_x else None, history=None,
                                 wall_time=max(q.wall_time for q in sols), **{f: cat([getattr(q, f) for q in sols]) for f in _SOL_FIELDS})
    out.solution._no_append = getattr(sols[0], "_no_append", False)
    if all(hasattr(q.lam, "is_complex") for q in parts):
        out.lam = cat([q.lam for q in parts])
    return out
