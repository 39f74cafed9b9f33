"""Tiled solver round loop: CUDA-graph replay vs stream launches (GPU dev tool).  Bitwise equality of
the results and solve timings for cfg4 (P pixels) and cfg5 (64 RHS), RBPG and FISTA."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200 import _lib
from paper_1805_01759_b200.synth import make_config

for cfg_id, P in ((5, 64), (4, int(os.environ.get("P4", "2048")))):
    batch = make_config(cfg_id, num_pixels=P)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    seeds = d.derive_seeds(2018, P)
    for be in ("rbpg", "fista"):
        cfg = tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8)
        out = {}
        for g in ("0", "1"):
            os.environ["TB_TILED_GRAPH"] = g
            r = d.solve(px, lam, cfg, be, seeds=seeds)
            torch.cuda.synchronize()
            ts = []
            for _ in range(2):
                l0 = _lib.launch_count()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); r = d.solve(px, lam, cfg, be, seeds=seeds); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
                nl = _lib.launch_count() - l0
            out[g] = (r, min(ts), nl)
        a, b = out["0"][0], out["1"][0]
        same = all(torch.equal(getattr(a, f), getattr(b, f)) for f in ("x_hat", "objective_final", "iterations", "status"))
        print(f"cfg{cfg_id} {be} P={P}: stream {out['0'][1]:.1f} ms ({out['0'][2]} launches)  graph {out['1'][1]:.1f} ms ({out['1'][2]} launches)  "
              f"bit-identical {same}  mean iters {a.iterations.double().mean().item():.1f}", flush=True)
