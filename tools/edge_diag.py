"""GPU vs oracle F histories on degenerate shapes (dev tool): first differing iteration per case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1805_01759_b200 as tb
from oracle import tomo_oracle as O

def rand(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)

rng = np.random.default_rng(11)
cases = [("n=1", rand(rng, (1, 30)), rand(rng, (3, 1)), 0.05, 1), ("m=1", rand(rng, (9, 1)), rand(rng, (3, 9)), 0.4, 1)]
rng2 = np.random.default_rng(3)
cases.append(("J=m", rand(rng2, (10, 24)), rand(rng2, (4, 10)), 0.3, 24))
for name, a, b, lam, J in cases:
    d = tb.Dictionary(a)
    for be in ("rbpg", "fista"):
        if be == "fista" and J > 1:
            continue
        cfg = tb.SolverConfig(max_iters=150, tol=1e-6, num_blocks=J)
        seeds = np.arange(1, b.shape[0] + 1, dtype=np.uint64) * 7919
        for path in ("auto", "tiled"):
            sol = d.solve(b, np.full(b.shape[0], lam), cfg, be, seeds=seeds, history=True, path=path)
            lips = d.partition(J).lipschitz if be == "rbpg" else d.lipschitz()
            for q in range(b.shape[0]):
                ref = O.SOLVERS[be](a.astype(np.complex128), b[q].astype(np.complex128), lam, O.SolverCfg(max_iters=150, tol=1e-6, num_blocks=J, seed=int(seeds[q])), lips)
                h = sol.history[q].cpu().numpy(); rh = ref["history"]
                k = min(len(rh), int(sol.iterations[q]) + 1)
                diff = np.abs(h[:k] - rh[:k]) / np.maximum(np.abs(rh[:k]), 1e-300)
                bad = np.flatnonzero(diff > 1e-9)
                first = int(bad[0]) if bad.size else -1
                print(f"{name} {be} {path} px{q}: iters gpu {int(sol.iterations[q])} ref {ref['iterations']}  first diff k={first}  "
                      + (f"gpu {h[first]:.10g} ref {rh[first]:.10g} prev gpu {h[first-1]:.10g} ref {rh[first-1]:.10g}" if first > 0 else ""), flush=True)
    print("lips", d.lipschitz(), 2 * O.spectral_sq_norm(a.astype(np.complex128)), d.partition(J).lipschitz[:4], O.block_lipschitz(a.astype(np.complex128), O.block_ranges(a.shape[1], J))[:4])
