"""Selection-kernel timing on the cfg2 batch (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config
b = make_config(2)
d = tb.Dictionary(b.dictionary)
px = torch.from_numpy(b.pixels).cuda()
lam = d.default_lambda(px, 0.1)
sol = d.solve(px, lam, tb.SolverConfig(max_iters=500, tol=1e-6, seed=2018), "rbpg", seeds=d.derive_seeds(2018, b.num_pixels))
est = tb.select_batch(d, sol.x_hat, px, b.grid, 2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    est = tb.select_batch(d, sol.x_hat, px, b.grid, 2)
e1.record(); torch.cuda.synchronize()
print(f"select_batch cfg2 1M px: {e0.elapsed_time(e1) / 5:.2f} ms; orders {torch.bincount(est.model_order.long()).tolist()}")
