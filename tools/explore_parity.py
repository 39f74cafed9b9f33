"""Exploratory GPU-vs-reference comparison on the golden cfg1 pixels (prints stats)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_01759_b200 import Dictionary, SolverConfig, PipelineConfig, select_batch
from paper_1805_01759_b200.grid import ParameterGrid

g = np.load("tests/golden/golden_v1.npz")
a = g["cfg1/a"]; pix = g["cfg1/b"]; lam = g["cfg1/lam"]; seeds = g["cfg1/pixel_seeds"]
d = Dictionary(a)
print("lip full", d.lipschitz(), float(g["cfg1/lip_full"]))
print("part8", d.partition(8).lipschitz - g["part8/lip"])
s = d.derive_seeds(2018, 24).cpu().numpy()
print("seeds equal", np.array_equal(s, seeds))
lt = d.default_lambda(pix, 0.1).cpu().numpy()
print("lambda rel", np.max(np.abs(lt - lam) / lam))
grid = ParameterGrid(elevation=g["cfg1/elev"])
for backend in ("rbpg", "fista", "ista"):
    cfg = SolverConfig(max_iters=500, tol=1e-6, num_blocks=8)
    t0 = time.time()
    bs = d.solve(pix, lam, cfg, backend, seeds=seeds, history=True)
    torch.cuda.synchronize()
    it = bs.iterations.cpu().numpy(); st = bs.status.cpu().numpy(); x = bs.x_hat.cpu().numpy(); ff = bs.objective_final.cpu().numpy()
    rit = g[f"cfg1/{backend}/iters"]; rst = g[f"cfg1/{backend}/status"]; rx = g[f"cfg1/{backend}/x"]
    rh = g[f"cfg1/{backend}/hist"]; rf = np.array([rh[p][rit[p]] for p in range(24)])
    xe = np.linalg.norm(x - rx, axis=1) / np.maximum(np.linalg.norm(rx, axis=1), 1e-30)
    print(backend, "time", time.time() - t0)
    print("  iters gpu", it); print("  iters ref", rit)
    print("  status eq", np.mean(st == rst), "F rel max", np.max(np.abs(ff - rf) / rf), "x relerr med/max", np.median(xe), xe.max())
    h = bs.history.cpu().numpy()
    k = min(50, int(it.min()))
    print("  hist rel (first 50) max", np.nanmax(np.abs(h[:, :k] - rh[:, :k]) / rh[:, :k]))
    est = select_batch(d, bs.x_hat, pix, grid, 2)
    sup = est.support.cpu().numpy(); rsup = g[f"cfg1/{backend}/support"]
    amps = est.amplitudes.cpu().numpy(); ramps = g[f"cfg1/{backend}/amps"]
    print("  support eq", np.mean(np.all(sup == rsup, axis=1)), "order eq", np.mean(est.model_order.cpu().numpy() == g[f"cfg1/{backend}/order"]))
    mask = np.abs(ramps) > 0
    print("  amp rel max", np.max(np.abs(amps - ramps)[mask] / np.abs(ramps)[mask]) if mask.any() else 0)
    sc = est.selection_scores.cpu().numpy(); rsc = g[f"cfg1/{backend}/scores"]
    print("  scores max abs diff", np.nanmax(np.abs(sc - rsc)))
