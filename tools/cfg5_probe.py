"""cfg5 tiled-path probe (single GPU): time per round for a backend."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config
backend = sys.argv[1] if len(sys.argv) > 1 else "rbpg"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c5 = make_config(5)
d = tb.Dictionary(c5.dictionary)
d.partition(8); d.lipschitz()
lam = d.default_lambda(c5.pixels, 0.1)
seeds = d.derive_seeds(2018, c5.num_pixels)
cfg = tb.SolverConfig(fixed_iters=iters, num_blocks=8)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    bs = d.solve(c5.pixels, lam, cfg, backend, seeds=seeds)
    torch.cuda.synchronize(); dt = time.time() - t0
    print(f"cfg5 {backend} iters={iters}: {dt*1000:.1f} ms, {dt/iters*1000:.2f} ms/round")
