import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config
c4 = make_config(4, num_pixels=256)
d = tb.Dictionary(c4.dictionary)
lam = d.default_lambda(c4.pixels, 0.1)
seeds = d.derive_seeds(2018, 256)
for be in ("fista", "rbpg"):
    for it in (5, 20, 100, 500):
        cfg = tb.SolverConfig(fixed_iters=it, num_blocks=8)
        r = d.solve(c4.pixels, lam, cfg, be, seeds=seeds)
        x = r.x_hat.cpu().numpy()
        nz = (x != 0)
        per = nz.sum(1)
        # union over 16-pixel groups per 64-col tile
        g = nz.reshape(16, 16, -1).any(1)  # [16 groups, m]
        t = g.reshape(16, -1, 64).any(2).mean()
        dens16 = g.mean()
        print(f"{be} it={it}: nnz/px median {np.median(per):.0f} max {per.max()} mean frac {per.mean()/x.shape[1]:.4f}; union-of-16 col density {dens16:.4f}; 64-col tiles touched {t:.3f}", flush=True)
