"""Solve-kernel timing of the library at TB_LIB_PATH (default: the in-tree build) on cfg1-3 (GPU dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config

RUNS = [(int(c), int(p), b) for c, p, b in (x.split(":") for x in os.environ.get("RUNS", "2:262144:rbpg,3:65536:rbpg,1:1024:rbpg").split(",") if x)]
for cfg_id, P, be in RUNS:
    batch = make_config(cfg_id, num_pixels=P)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    seeds = d.derive_seeds(2018, P)
    cfg = tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8)
    r = d.solve(px, lam, cfg, be, seeds=seeds)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = d.solve(px, lam, cfg, be, seeds=seeds); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    its = r.iterations.double().sum().item()
    flop = 16.0 * batch.n * batch.m / (8 if be == "rbpg" else 1)
    print(f"{os.path.basename(os.environ.get('TB_LIB_PATH', 'default'))} cfg{cfg_id} {be} P={P}: {ms:.2f} ms  {P / ms * 1e3 / 1e6:.4f} M px/s  {its * flop / ms / 1e9 / 70.78:.4f} of FP32  iters {its:.0f}", flush=True)
