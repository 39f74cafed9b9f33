"""Multi-GPU host logic on CPU: pixel shards, RBPG block striping, and the column-sharded
reduction plumbing exercised with a real 2-process gloo all-reduce (no GPU needed)."""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import tomo_oracle as O
from paper_1805_01759_b200.sharded import column_shards, gather_columns, local_columns, pixel_shard


@pytest.mark.parametrize("p,w", [(10, 1), (10, 3), (1 << 20, 8), (5, 8)])
def test_pixel_shards_partition(p, w):
    spans = [pixel_shard(p, w, g) for g in range(w)]
    assert spans[0][0] == 0 and spans[-1][1] == p
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    sizes = [e - s for s, e in spans]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("m,w,j", [(300, 2, 8), (1 << 20, 8, 8), (160000, 4, 8), (1000, 3, None)])
def test_column_shards_cover_each_column_once(m, w, j):
    shards = column_shards(m, w, j)
    cols = np.sort(np.concatenate([local_columns(r) for r in shards]))
    np.testing.assert_array_equal(cols, np.arange(m))
    if j is not None:
        # rank g's local block b is a stripe of the reference block b (solver.py:204-210)
        for b, (s, e) in enumerate(O.block_ranges(m, j)):
            stripes = [shards[g][b] for g in range(w)]
            assert stripes[0][0] == s and stripes[-1][1] == e
            assert all(x[1] == y[0] for x, y in zip(stripes, stripes[1:]))


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    n, m, p = 7, 64, 5
    a = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
    z = (rng.standard_normal((p, m)) + 1j * rng.standard_normal((p, m))) * (rng.random((p, m)) < 0.2)
    ranges = column_shards(m, world, 4)[rank]
    cols = local_columns(ranges)
    # the per-shard "red" buffer layout: [P][n] complex forward partial, then [P][4] scalars
    part = z[:, cols] @ a[:, cols].T
    sc = np.stack([np.sum(np.abs(z[:, cols]) ** 2, axis=1), np.sum(np.abs(z[:, cols]), axis=1), np.zeros(p), np.zeros(p)], axis=1)
    red = torch.from_numpy(np.concatenate([part.view(np.float64).reshape(-1), sc.reshape(-1)]))
    dist.all_reduce(red)
    full = red.numpy()
    got = full[: p * n * 2].view(np.complex128).reshape(p, n)
    ok = np.allclose(got, z @ a.T, rtol=1e-12, atol=1e-12) and np.allclose(full[p * n * 2 :].reshape(p, 4)[:, 1], np.abs(z).sum(axis=1))
    xs = gather_columns([z[:, local_columns(column_shards(m, world, 4)[g])].astype(np.complex64) for g in range(world)], column_shards(m, world, 4), m)
    ok = ok and np.array_equal(xs, z.astype(np.complex64))
    out[rank] = int(ok)
    dist.barrier()
    dist.destroy_process_group()


def test_column_sharded_reduction_gloo_world2():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert dict(out) == {0: 1, 1: 1}


def _gather_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_1805_01759_b200.sharded import gather_estimates
    from paper_1805_01759_b200.slimmer import BatchEstimates
    from paper_1805_01759_b200.solver import BatchSolution

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, k = 7, 2
    s, e = pixel_shard(p, world, rank)
    ids = torch.arange(s, e)
    est = BatchEstimates(
        model_order=ids.to(torch.int32), support=torch.stack([ids, -ids], 1), amplitudes=(ids[:, None] * (1 + 2j)).repeat(1, k).to(torch.complex128),
        elevations=ids[:, None].double().repeat(1, k), motion_params=torch.zeros(e - s, k, 0, dtype=torch.float64),
        selection_scores=ids[:, None].double().repeat(1, k + 1), n_scores=ids.to(torch.int32), error=torch.zeros(e - s, dtype=torch.int32),
    )
    est.solution = BatchSolution(x_hat=(ids[:, None] * 1j).repeat(1, 3).to(torch.complex64), objective_final=ids.double(), iterations=ids.to(torch.int32), status=ids.to(torch.int32) % 4)
    full = gather_estimates(est, p)
    want = torch.arange(p)
    ok = torch.equal(full.model_order, want.to(torch.int32)) and torch.equal(full.support[:, 1], -want)
    ok = ok and torch.equal(full.amplitudes[:, 0], (want * (1 + 2j)).to(torch.complex128)) and torch.equal(full.solution.x_hat[:, 2], (want * 1j).to(torch.complex64))
    ok = ok and torch.equal(full.solution.objective_final, want.double()) and full.motion_params.shape == (p, k, 0)
    out[rank] = int(ok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_estimates_ordered_gloo(world):
    """Ordered all-gather of ragged contiguous pixel shards (7 pixels over 2 or 3 ranks)."""
    port = 29700 + (os.getpid() % 200) + world
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, port, out), nprocs=world, join=True)
    assert dict(out) == {g: 1 for g in range(world)}
