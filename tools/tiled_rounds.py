"""A short tiled solve for an ncu launch list (GPU dev tool): CFG=5 BACKEND=rbpg ITERS=20 P=64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config

cfg_id, P = int(os.environ.get("CFG", "5")), int(os.environ.get("P", "64"))
be, iters = os.environ.get("BACKEND", "rbpg"), int(os.environ.get("ITERS", "20"))
batch = make_config(cfg_id, num_pixels=P)
d = tb.Dictionary(batch.dictionary)
px = torch.from_numpy(batch.pixels).cuda()
lam = d.default_lambda(px, 0.1)
seeds = d.derive_seeds(2018, P)
if be == "rbpg":
    d.partition(8)
else:
    d.lipschitz()
torch.cuda.synchronize()
os.environ["TB_TILED_GRAPH"] = "0"
r = d.solve(px, lam, tb.SolverConfig(fixed_iters=iters, num_blocks=8), be, seeds=seeds)
torch.cuda.synchronize()
