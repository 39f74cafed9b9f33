"""One solve launch for ncu (GPU dev tool): PREC=fp64|c64 CFG=2 P=65536 BACKEND=rbpg."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config

cfg_id, P = int(os.environ.get("CFG", "2")), int(os.environ.get("P", "65536"))
prec, be = os.environ.get("PREC", "c64"), os.environ.get("BACKEND", "rbpg")
batch = make_config(cfg_id, num_pixels=P)
d = tb.Dictionary(batch.dictionary)
px = torch.from_numpy(batch.pixels).cuda()
lam = d.default_lambda(px, 0.1)
seeds = d.derive_seeds(2018, P)
cfg = tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018)
r = d.solve(px, lam, cfg, be, seeds=seeds)
torch.cuda.synchronize()
print("mean iters", r.iterations.double().mean().item())
