"""Throughput of the batched Monte-Carlo harness: realizations/s, host synthesis vs device.

usage: python tools/mc_bench.py [realizations_per_cell] [workers] [--reference]
With --reference (build container only: imports /root/reference) it times the reference harness on
a bounded sample instead (first cell-major slice of the same tasks, process pool of `workers`).
"""
import json
import os
import sys
import time

if "--reference" in sys.argv:  # one BLAS thread per worker process (set before numpy loads)
    os.environ["OPENBLAS_NUM_THREADS"] = os.environ["OMP_NUM_THREADS"] = "1"

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
W = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
KAPPAS, SNRS, METHODS = [0.4, 0.8, 1.2], [5.0, 10.0, 20.0], ["rbpg", "fista", "svd_wiener"]

if "--reference" in sys.argv:
    sys.path.insert(0, "/root/reference/pkg/src")
    from tomobpdn import simulate as RS
    from tomobpdn.solver import SolverConfig as RC

    base = RS.Scenario(geometry=RS.demo_geometry(), seed=7)
    setup = RS.MonteCarloSetup(solver=RC(max_iters=500, tol=1e-6))
    t0 = time.time()
    res = RS.monte_carlo_detection(base, KAPPAS, SNRS, METHODS, R, setup, workers=W)
    dt = time.time() - t0
    n = len(KAPPAS) * len(SNRS) * len(METHODS) * R
    print(json.dumps({"impl": "reference", "realizations": n, "seconds": dt, "realizations_per_s": n / dt, "workers": W}))
    sys.exit(0)

import torch  # noqa: E402
from paper_1805_01759_b200 import simulate as S  # noqa: E402
from paper_1805_01759_b200.solver import SolverConfig  # noqa: E402

base = S.Scenario(geometry=S.demo_geometry(), seed=7)
setup = S.MonteCarloSetup(solver=SolverConfig(max_iters=500, tol=1e-6))
grid = S.harness_grid(base, setup)
cells = [(k, s, m) for k in KAPPAS for s in SNRS for m in METHODS]
items = [(cells[c][0], cells[c][1], c * R + r) for c in range(len(cells)) for r in range(R)]
S.monte_carlo_detection(base, KAPPAS, SNRS, METHODS, 8, setup)  # warm-up (library load, contexts)
torch.cuda.synchronize()
t0 = time.time()
S._draw_all(base, grid, setup, items, W)
t_host = time.time() - t0
t0 = time.time()
res = S.monte_carlo_detection(base, KAPPAS, SNRS, METHODS, R, setup, workers=W)
torch.cuda.synchronize()
dt = time.time() - t0
n = len(items)
print(json.dumps({"impl": "b200", "draws": "host", "realizations": n, "seconds": dt, "realizations_per_s": n / dt, "host_synthesis_s": t_host,
                  "workers": W, "p_d": {f"{r.kappa}/{r.snr_db}/{r.method}": r.p_d for r in res}}))
S.monte_carlo_detection(base, KAPPAS, SNRS, METHODS, 8, setup, draws="device")  # warm-up
torch.cuda.synchronize()
t0 = time.time()
res2 = S.monte_carlo_detection(base, KAPPAS, SNRS, METHODS, R, setup, draws="device")
torch.cuda.synchronize()
dt2 = time.time() - t0
print(json.dumps({"impl": "b200", "draws": "device", "realizations": n, "seconds": dt2, "realizations_per_s": n / dt2,
                  "p_d": {f"{r.kappa}/{r.snr_db}/{r.method}": r.p_d for r in res2}}))
