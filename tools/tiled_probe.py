"""Small cfg4 tiled-path run for launch-list profiling."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config
backend = sys.argv[1] if len(sys.argv) > 1 else "rbpg"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 512
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
c4 = make_config(4, num_pixels=P)
d = tb.Dictionary(c4.dictionary)
d.partition(8); d.lipschitz()
lam = d.default_lambda(c4.pixels, 0.1)
seeds = d.derive_seeds(2018, P)
cfg = tb.SolverConfig(fixed_iters=iters, num_blocks=8)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    bs = d.solve(c4.pixels, lam, cfg, backend, seeds=seeds)
    torch.cuda.synchronize(); dt = time.time() - t0
    print(f"tc={os.environ.get('TB_TILED_TC','-')} F={float(bs.objective_final.double().sum()):.12e} {backend} P={P} iters={iters}: {dt*1000:.1f} ms, {dt/iters*1000:.2f} ms/round, {P*iters*16*100*160000/(8 if backend=='rbpg' else 1)/dt/1e12:.2f} TF/s")
