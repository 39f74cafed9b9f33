"""Multi-process paths through the REAL library: two ranks (processes) on the one GPU this
environment provides, over a gloo process group.  The ranks never wait on each other inside a
kernel -- every exchange is a host-side collective between kernel launches -- so sharing one GPU
changes only the timing, not the algorithm.

* pixel sharding (cfg1-4): ``pipeline_sharded`` and the distributed
  ``solve_stack`` give byte-identical results for world size 1 and 2 (the reference's worker-count
  invariance, test_acceptance.py:266-312 / test_cli.py:123-131);
* column sharding (cfg5): ``solve_column_sharded`` with ``reduce_fn = dist.all_reduce`` on the
  per-round CUDA ``red`` buffers equals the unsharded solve exactly.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.multiprocessing as mp  # noqa: E402


def _init(rank, world, port):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _pixel_worker(rank, world, port, out, stack_bytes, grid_json):
    import json

    dist = _init(rank, world, port)
    import paper_1805_01759_b200 as tb
    from paper_1805_01759_b200.stack import solve_stack
    from paper_1805_01759_b200.synth import make_config

    batch = make_config(1, num_pixels=257)
    res = {}
    for backend in ("rbpg", "fista"):
        pc = tb.PipelineConfig(solver=tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018), backend=backend, k_max=2)
        est = tb.pipeline_sharded(batch.dictionary, batch.pixels, batch.grid, pc, beta=0.1)
        res[backend] = {f: getattr(est, f).cpu().numpy() for f in ("model_order", "support", "amplitudes", "selection_scores")}
        res[backend].update({f: getattr(est.solution, f).cpu().numpy() for f in ("objective_final", "iterations", "status", "x_hat")})
    path = f"/tmp/tb_mp_{port}_{world}_{rank}.tstk"
    with open(path, "wb") as fh:
        fh.write(stack_bytes)
    cfg = tb.PipelineConfig(solver=tb.SolverConfig(max_iters=500, tol=1e-6), backend="rbpg", k_max=2)
    outp = f"/tmp/tb_mp_{port}_{world}.jsonl"
    solve_stack(path, json.loads(grid_json), cfg, out_jsonl=outp if rank == 0 else None)
    dist.barrier()
    if rank == 0:
        with open(outp, "rb") as fh:
            res["jsonl"] = fh.read()
        out["w"] = res
    dist.destroy_process_group()


def _spawn(fn, world, *args):
    port = 29000 + (os.getpid() * 7 + world) % 2000
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(fn, args=(world, port, out) + args, nprocs=world, join=True)
    return dict(out)


@pytest.fixture(scope="module")
def stack_case(golden):
    return golden["cli/stack"].tobytes(), str(golden["cli/g1"])


def test_pixel_sharded_world1_vs_world2_bitwise(stack_case):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    one = _spawn(_pixel_worker, 1, *stack_case)["w"]
    two = _spawn(_pixel_worker, 2, *stack_case)["w"]
    for backend in ("rbpg", "fista"):
        for f, v in one[backend].items():
            assert v.dtype == two[backend][f].dtype and np.array_equal(v, two[backend][f], equal_nan=True), (backend, f)
    assert one["jsonl"] == two["jsonl"] and len(one["jsonl"]) > 0


def _column_worker(rank, world, port, out):
    dist = _init(rank, world, port)
    import paper_1805_01759_b200 as tb
    from paper_1805_01759_b200.sharded import ColumnShard, column_shards, local_columns, solve_column_sharded
    from paper_1805_01759_b200.synth import motion_dictionary

    rng = np.random.default_rng(21)
    freqs, times = np.sort(rng.uniform(-0.5, 0.5, 100)), np.sort(rng.uniform(0, 4, 100))
    grid = tb.ParameterGrid(elevation=(np.arange(64) - 32) * 0.25, motion_axes=(np.linspace(-0.02, 0.02, 16), np.linspace(0, 0.01, 8)), motion_bases=("linear", "seasonal"))
    a = motion_dictionary(freqs, times, grid).astype(np.complex64)
    pos = rng.integers(0, a.shape[1], (6, 3))
    a128 = a.astype(np.complex128)
    b = sum(a128[:, pos[:, k]].T * (1.0 - 0.2 * k) for k in range(3))
    b = (b + 0.2 * (rng.standard_normal(b.shape) + 1j * rng.standard_normal(b.shape))).astype(np.complex64)
    res = {}
    for backend in ("rbpg", "fista"):
        full = tb.Dictionary(a)
        lam = full.default_lambda(b, 0.1)
        seeds = full.derive_seeds(5, b.shape[0])
        lips = full.partition(8).lipschitz if backend == "rbpg" else full.lipschitz()
        cfg = tb.SolverConfig(max_iters=120, tol=1e-6, num_blocks=8)
        ranges = column_shards(a.shape[1], world, 8 if backend == "rbpg" else None)[rank]
        shard = ColumnShard(a[:, local_columns(ranges)], ranges, backend, 8, lips)
        sol = solve_column_sharded([shard], b, lam, cfg, seeds=seeds, reduce_fn=lambda bufs: dist.all_reduce(bufs[0]), history=True)[0]
        ref = full.solve(b, lam, cfg, backend, seeds=seeds, history=True, path="tiled")
        res[backend] = dict(
            its=bool(torch.equal(sol.iterations, ref.iterations)), st=bool(torch.equal(sol.status, ref.status)),
            f=float((sol.objective_final - ref.objective_final).abs().max() / ref.objective_final.abs().max()),
            hist=bool(torch.allclose(sol.history, ref.history, rtol=1e-9, atol=0.0, equal_nan=True)),
            x=float((sol.x_hat.cpu() - ref.x_hat.cpu()[:, local_columns(ranges)]).abs().max()),
        )
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_column_sharded_gloo_allreduce_world2():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    res = _spawn(_column_worker, 2)
    for rank in (0, 1):
        for backend in ("rbpg", "fista"):
            r = res[rank][backend]
            assert r["its"] and r["st"] and r["hist"], (rank, backend, r)
            assert r["f"] <= 1e-10 and r["x"] <= 1e-6, (rank, backend, r)
