"""Generate tests/golden/golden_large_v1.npz: BASELINE cfg4 and cfg5 solved by the REAL reference.

Run in the build container (the reference is importable there, not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_large.py

cfg4 (n=100, m=160,000): 8 pixels sampled across the 16,384-pixel batch, FISTA and RBPG at the
BASELINE settings (max_iters=500, tol=1e-6), then the reference's own selection
(slimmer.py:77-190, k_max=2, p = 3 + 2 motion axes).
cfg5 (n=100, m=1,048,576): 2 right-hand sides, FISTA and RBPG with fixed_iters=60, RBPG at
max_iters=500 / tol=1e-6 to convergence, selection with k_max=3 on the converged RBPG x_hat.

Inputs are the package's seeded synthesis (``synth.make_config``): A and b rounded to complex64
once, lambda = 0.1 max|A^H b| rounded to float32 (host fp64), pixel seeds by the cli.py:102 rule.
The dictionaries are too large to commit (128 MB / 800 MiB); the fixture stores the SHA-256 of
the complex64 dictionary bytes so the GPU test proves it rebuilt the identical matrix.
The reference's per-solve setup (spectral_sq_norm / block_partition) runs exactly as shipped:
no Lipschitz constant is passed in.  x_hat is stored sparsely (indices + values of the nonzeros).
The reference's own wall times per solve are recorded as well (single core, BLAS 1 thread).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

STATUS = {"converged": 0, "max-iters": 1, "line-search-failure": 2, "numerical-failure": 3}
CFG4_PIXELS = [0, 1, 2, 3, 5000, 9999, 12345, 16383]
CFG5_RHS = [0, 41]
RUN_SEED = 2018
PARTS = "/tmp/golden_large_parts"

_STATE = {}


def _load(cfg):
    if cfg not in _STATE:
        from paper_1805_01759_b200.synth import lambda_from_beta, make_config

        batch = make_config(cfg)
        ids = CFG4_PIXELS if cfg == 4 else CFG5_RHS
        pix = batch.pixels[ids]
        lam = lambda_from_beta(batch.dictionary, pix, 0.1)
        a = batch.dictionary.astype(np.complex128)
        _STATE[cfg] = (batch, ids, pix, lam, a)
    return _STATE[cfg]


def task(spec):
    cfg, j, backend, mode = spec
    name = f"cfg{cfg}_{j}_{backend}_{mode}"
    out = os.path.join(PARTS, name + ".npz")
    if os.path.exists(out):
        return name
    import tomobpdn as T
    from tomobpdn.rng import derive_seed, substream

    batch, ids, pix, lam, a = _load(cfg)
    pid = ids[j]
    seed = derive_seed(substream(RUN_SEED, pid))
    if mode == "conv":
        sc = T.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=int(seed))
    else:
        sc = T.SolverConfig(fixed_iters=int(mode[5:]), tol=1e-6, num_blocks=8, seed=int(seed))
    obj = T.Objective(dictionary=a, measurement=pix[j].astype(np.complex128), lambda_reg=float(lam[j]))
    t0 = time.perf_counter()
    sol = {"rbpg": T.rbpg_solve, "fista": T.fista_solve}[backend](obj, sc)
    wall = time.perf_counter() - t0
    res = {
        "seed": np.uint64(seed),
        "iters": sol.iterations_used,
        "status": STATUS[sol.status.value],
        "hist": sol.objective_history,
        "wall": wall,
    }
    nz = np.flatnonzero(sol.x_hat)
    res["x_idx"] = nz
    res["x_val"] = sol.x_hat[nz]
    res["x_norm"] = np.linalg.norm(sol.x_hat)
    if mode == "conv":
        grid = T.ParameterGrid(elevation=batch.grid.elevation, motion_axes=batch.grid.motion_axes, motion_bases=batch.grid.motion_bases)
        k_max = batch.k_max
        from tomobpdn import slimmer

        cands = slimmer.detect_support(sol.x_hat, grid, k_max)
        k_hat, support, scores = slimmer.model_select(obj, cands, k_max, 3 + len(grid.motion_axes))
        e = slimmer.estimate_params(obj, grid, support)
        res["cands"] = np.asarray(cands)
        res["order"] = k_hat
        res["support"] = np.asarray(support)
        res["amps"] = np.asarray(e.amplitudes)
        res["elevs"] = np.asarray(e.elevations)
        res["motion"] = np.asarray(e.motion_params)
        res["scores"] = np.asarray(scores)
    np.savez(out + ".tmp.npz", **res)
    os.replace(out + ".tmp.npz", out)
    print(f"{name}: iters={sol.iterations_used} status={sol.status.value} wall={wall:.1f}s nnz={nz.size}", flush=True)
    return name


def main():
    from concurrent.futures import ProcessPoolExecutor

    os.makedirs(PARTS, exist_ok=True)
    t5 = [(5, j, b, m) for j in range(len(CFG5_RHS)) for b, m in (("fista", "fixed60"), ("rbpg", "fixed60"), ("rbpg", "conv"))]
    t4 = [(4, j, b, "conv") for j in range(len(CFG4_PIXELS)) for b in ("fista", "rbpg")]
    workers = int(os.environ.get("GOLDEN_WORKERS", "4"))
    with ProcessPoolExecutor(len(t5)) as p5, ProcessPoolExecutor(workers) as p4:
        f5 = [p5.submit(task, t) for t in t5]
        f4 = [p4.submit(task, t) for t in t4]
        for f in f4 + f5:
            f.result()

    from paper_1805_01759_b200.synth import make_config

    out = {}
    for cfg, ids in ((4, CFG4_PIXELS), (5, CFG5_RHS)):
        batch = make_config(cfg, num_pixels=max(ids) + 1)
        from paper_1805_01759_b200.synth import lambda_from_beta

        pix = batch.pixels[ids]
        out[f"cfg{cfg}/ids"] = np.array(ids)
        out[f"cfg{cfg}/b"] = pix
        out[f"cfg{cfg}/lam"] = lambda_from_beta(batch.dictionary, pix, 0.1)
        out[f"cfg{cfg}/a_sha256"] = np.array(hashlib.sha256(np.ascontiguousarray(batch.dictionary).tobytes()).hexdigest())
        out[f"cfg{cfg}/a_shape"] = np.array(batch.dictionary.shape)
    for fn in sorted(os.listdir(PARTS)):
        if not fn.endswith(".npz") or ".tmp" in fn:
            continue
        cfg_j_b_m = fn[:-4]
        cfgs, j, b, m = cfg_j_b_m.split("_")
        d = np.load(os.path.join(PARTS, fn))
        for k in d.files:
            out[f"{cfgs}/{b}_{m}/{j}/{k}"] = d[k]
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_large_v1.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
