"""Dev tool (build container only: reads /root/reference): speed and iteration agreement of the
real reference solvers vs the oracle port on the first 24 cfg2 pixels, one core."""
import os, sys, time
os.environ["OPENBLAS_NUM_THREADS"] = "1"; os.environ["OMP_NUM_THREADS"] = "1"
sys.path.insert(0, "/root/reference/pkg/src"); sys.path.insert(0, "/root/repo")
import numpy as np
import tomobpdn
from tomobpdn import solver as RS, prox as RP
from oracle import tomo_oracle as O
from paper_1805_01759_b200.synth import make_config, lambda_from_beta
b = make_config(2, num_pixels=24)
a = b.dictionary.astype(np.complex128)
lam = lambda_from_beta(b.dictionary, b.pixels, 0.1)
seeds = [O.derive_seed(2018, p) for p in range(24)]
for backend in ("rbpg", "fista"):
    t0 = time.perf_counter(); its_r = []
    for p in range(24):
        obj = RP.Objective(a, b.pixels[p].astype(np.complex128), float(lam[p]))
        cfg = RS.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=int(seeds[p]))
        sol = (RS.rbpg_solve if backend == "rbpg" else RS.fista_solve)(obj, cfg)
        its_r.append(sol.iterations_used)
    tr = time.perf_counter() - t0
    t0 = time.perf_counter(); its_o = []
    for p in range(24):
        cfg = O.SolverCfg(max_iters=500, tol=1e-6, num_blocks=8, seed=int(seeds[p]))
        sol = O.SOLVERS[backend](a, b.pixels[p].astype(np.complex128), float(lam[p]), cfg)
        its_o.append(sol["iterations"])
    to = time.perf_counter() - t0
    print(f"{backend}: reference {24/tr:.1f} px/s/core, oracle port {24/to:.1f} px/s/core, iterations equal {its_r == its_o}")
