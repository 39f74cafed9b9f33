"""Process-pool driver over the CPU oracle -- TEST / BASELINE INFRASTRUCTURE ONLY.

Mirrors the reference's own parallel pattern (cli.py:136-144: ProcessPoolExecutor, the
dictionary shipped once through the pool initializer, pixels chunked, output order pinned by
map) so ``bench.py`` can time the reference algorithm on all host cores and the tests can
build per-pixel expectations for large samples.
"""

from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from . import tomo_oracle as O

_STATE: dict = {}


def _init(a, grid_desc, backend, cfg_kw, lips, k_max, pin_blas):
    if pin_blas:
        for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[var] = "1"
        try:
            from threadpoolctl import threadpool_limits

            threadpool_limits(1)
        except Exception:
            pass
    _STATE.update(a=np.asarray(a, dtype=complex), grid=grid_desc, backend=backend, cfg_kw=cfg_kw, lips=lips, k_max=k_max)


class GridDesc:
    """Picklable grid description with the attributes the oracle reads."""

    def __init__(self, elevation, motion_axes=()):
        self.elevation = np.asarray(elevation, dtype=float)
        self.motion_axes = tuple(np.asarray(x, dtype=float) for x in motion_axes)
        self.shape = (self.elevation.size,) + tuple(x.size for x in self.motion_axes)


def _work(task):
    b, lam, seed, want_x = task
    st = _STATE
    cfg = O.SolverCfg(seed=int(seed), **st["cfg_kw"])
    if st["grid"] is None:
        sol = O.SOLVERS[st["backend"]](st["a"], np.asarray(b, dtype=complex), float(lam), cfg, st["lips"])
        return {"iterations": sol["iterations"], "status": sol["status"], "f_final": float(sol["history"][-1]), "x_hat": sol["x_hat"] if want_x else None}
    est = O.pipeline(st["a"], np.asarray(b, dtype=complex), float(lam), st["grid"], st["k_max"], st["backend"], cfg, st["lips"])
    sol = est.pop("solution")
    est.update(iterations=sol["iterations"], status=sol["status"], f_final=float(sol["history"][-1]), x_hat=sol["x_hat"] if want_x else None)
    return est


def run(a, pixels, lam, backend, seeds=None, grid=None, k_max=2, workers=None, lips=None, want_x=False, chunksize=8, pin_blas=True, **cfg_kw):
    """Solve (and, with ``grid``, run the pipeline on) every pixel with the oracle; ordered results."""
    p = len(pixels)
    seeds = np.zeros(p, dtype=np.uint64) if seeds is None else np.asarray(seeds, dtype=np.uint64)
    tasks = [(pixels[i], float(lam[i]), int(seeds[i]), want_x) for i in range(p)]
    workers = workers or os.cpu_count() or 1
    args = (a, grid, backend, cfg_kw, lips, k_max, pin_blas)
    if workers == 1:
        _init(*args)
        return [_work(t) for t in tasks]
    with ProcessPoolExecutor(max_workers=workers, initializer=_init, initargs=args) as pool:
        return list(pool.map(_work, tasks, chunksize=chunksize))
