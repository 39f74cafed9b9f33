import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config
batch = make_config(1); P = batch.num_pixels
d = tb.Dictionary(batch.dictionary); pix = torch.from_numpy(batch.pixels).cuda()
scfg = tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018)
pcfg = tb.PipelineConfig(solver=scfg, backend="rbpg", k_max=2)
for _ in range(3): tb.pipeline_batch(d, pix, batch.grid, pcfg, beta=0.1)
torch.cuda.synchronize()
T = {}
def t(name, f):
    t0 = time.perf_counter(); r = f(); T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    lam = t("lambda", lambda: d.default_lambda(pix, 0.1))
    seeds = t("seeds", lambda: d.derive_seeds(2018, P, 0))
    sol = t("solve", lambda: d.solve(pix, lam, scfg, "rbpg", seeds=seeds))
    est = t("select", lambda: tb.select_batch(d, sol.x_hat, pix, batch.grid, 2))
e1.record(); torch.cuda.synchronize()
print("device ms/step", e0.elapsed_time(e1) / 10, {k: round(v * 100, 3) for k, v in T.items()}, "ms/step host")
e0.record()
for _ in range(10):
    est = t("pipeline", lambda: tb.pipeline_batch(d, pix, batch.grid, pcfg, beta=0.1))
e1.record(); torch.cuda.synchronize()
print("pipeline device ms/step", e0.elapsed_time(e1) / 10, round(T["pipeline"] * 100, 3))
