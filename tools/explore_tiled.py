"""Exploratory checks of the tiled large-dictionary path (prints stats)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_01759_b200 import Dictionary, SolverConfig, select_batch, ParameterGrid
from paper_1805_01759_b200.synth import motion_dictionary, make_config, lambda_from_beta
from oracle import tomo_oracle as O
from oracle import batch as OB

g = np.load("tests/golden/golden_v1.npz")
a = g["cfg1/a"]; pix = g["cfg1/b"]; lam = g["cfg1/lam"]; seeds = g["cfg1/pixel_seeds"]
d = Dictionary(a)
for backend in ("rbpg", "fista", "ista"):
    cfg = SolverConfig(max_iters=500, tol=1e-6, num_blocks=8)
    t0 = time.time()
    bs = d.solve(pix, lam, cfg, backend, seeds=seeds, history=True, path="tiled")
    torch.cuda.synchronize()
    it = bs.iterations.cpu().numpy(); st = bs.status.cpu().numpy(); x = bs.x_hat.cpu().numpy(); ff = bs.objective_final.cpu().numpy()
    rit = g[f"cfg1/{backend}/iters"]; rst = g[f"cfg1/{backend}/status"]; rx = g[f"cfg1/{backend}/x"]
    rh = g[f"cfg1/{backend}/hist"]; rf = np.array([rh[p][rit[p]] for p in range(24)])
    xe = np.linalg.norm(x - rx, axis=1) / np.maximum(np.linalg.norm(rx, axis=1), 1e-30)
    print(f"tiled cfg1 {backend}: {time.time()-t0:.2f}s iters_eq {np.mean(it==rit):.3f} status_eq {np.mean(st==rst):.3f} Frel {np.max(np.abs(ff-rf)/rf):.2e} x med/max {np.median(xe):.2e}/{xe.max():.2e}")

# mid-size motion grid, tiled vs oracle
rng = np.random.default_rng(5)
freqs = np.sort(rng.uniform(-0.5, 0.5, 100)); times = np.sort(rng.uniform(0, 4, 100))
grid = ParameterGrid(elevation=(np.arange(40) - 20) * 0.25, motion_axes=(np.linspace(-0.02, 0.02, 10), np.linspace(0, 0.01, 10)), motion_bases=("linear", "seasonal"))
A = motion_dictionary(freqs, times, grid).astype(np.complex64)
m = A.shape[1]
P = 16
pos = rng.integers(0, m, (P, 2))
B = (A.astype(np.complex128)[:, pos[:, 0]].T + 0.7 * A.astype(np.complex128)[:, pos[:, 1]].T)
B = (B + 0.3 * (rng.standard_normal(B.shape) + 1j * rng.standard_normal(B.shape))).astype(np.complex64)
dm = Dictionary(A)
lamm = dm.default_lambda(B, 0.1).cpu().numpy()
sd = dm.derive_seeds(3, P).cpu().numpy()
for backend in ("rbpg", "fista"):
    cfg = SolverConfig(max_iters=80, tol=1e-6, num_blocks=8)
    t0 = time.time()
    bs = dm.solve(B, lamm, cfg, backend, seeds=sd, path="tiled")
    torch.cuda.synchronize(); tg = time.time() - t0
    lips = dm.partition(8).lipschitz if backend == "rbpg" else dm.lipschitz()
    t0 = time.time()
    ref = OB.run(A.astype(np.complex128), B, lamm, backend, seeds=sd, lips=lips, want_x=True, max_iters=80, tol=1e-6, num_blocks=8)
    to = time.time() - t0
    it = bs.iterations.cpu().numpy(); ff = bs.objective_final.cpu().numpy(); x = bs.x_hat.cpu().numpy()
    rit = np.array([r["iterations"] for r in ref]); rf = np.array([r["f_final"] for r in ref]); rx = np.array([r["x_hat"] for r in ref])
    xe = np.linalg.norm(x - rx, axis=1) / np.maximum(np.linalg.norm(rx, axis=1), 1e-30)
    print(f"mid m={m} {backend}: gpu {tg:.2f}s oracle {to:.1f}s iters_eq {np.mean(it==rit):.3f} Frel {np.max(np.abs(ff-rf)/rf):.2e} x med/max {np.median(xe):.2e}/{xe.max():.2e}")
    # auto path (tb_solve -> tiled in C++)
    bs2 = dm.solve(B, lamm, cfg, backend, seeds=sd)
    print("   auto==tiled", torch.equal(bs2.objective_final, bs.objective_final), torch.equal(bs2.iterations, bs.iterations))

# cfg4 timing
t0 = time.time(); c4 = make_config(4, num_pixels=int(os.environ.get("C4P", "512"))); print("cfg4 synth", time.time() - t0)
d4 = Dictionary(c4.dictionary)
t0 = time.time(); d4.partition(8); d4.lipschitz(); torch.cuda.synchronize(); print("cfg4 power iterations", time.time() - t0)
lam4 = d4.default_lambda(c4.pixels, 0.1)
for backend in ("rbpg", "fista"):
    cfg = SolverConfig(max_iters=500, tol=1e-6, num_blocks=8)
    t0 = time.time()
    bs = d4.solve(c4.pixels, lam4, cfg, backend, seeds=d4.derive_seeds(2018, c4.num_pixels))
    torch.cuda.synchronize(); tg = time.time() - t0
    it = bs.iterations.cpu().numpy(); st = bs.status.cpu().numpy()
    est = select_batch(d4, bs.x_hat, c4.pixels, c4.grid, 2)
    sup = est.support.cpu().numpy()
    hit = np.mean([set(int(v) for v in sup[p] if v >= 0) == set(c4.truth_support[p]) for p in range(c4.num_pixels)])
    pi = float(it.sum())
    print(f"cfg4 {backend}: {c4.num_pixels} px in {tg:.2f}s -> {c4.num_pixels/tg:.1f} px/s; mean iters {it.mean():.0f}; conv {np.mean(st==0):.2f}; truth-support hit {hit:.2f}; {pi*16*100*160000/(8 if backend=='rbpg' else 1)/tg/1e12:.2f} TFLOP/s algorithmic")
