"""Warp-solver iteration check (GPU): per-pixel iteration/status agreement with the oracle on cfg2/cfg3
subsets, plus solve-kernel timing at a larger batch.  Development tool, prints a summary."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config
from oracle import batch as OB

npx_chk = int(os.environ.get("CHK_PX", "256"))
for cfg_id, backends in (((2, ("rbpg", "fista")), (3, ("rbpg", "fista"))) if npx_chk else ()):
    batch = make_config(cfg_id, num_pixels=npx_chk)
    d = tb.Dictionary(batch.dictionary)
    a = batch.dictionary.astype(np.complex128)
    lam = d.default_lambda(batch.pixels, 0.1)
    seeds = d.derive_seeds(2018, npx_chk)
    for be in backends:
        cfg = tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018)
        r = d.solve(batch.pixels, lam, cfg, be, seeds=seeds)
        lips = d.partition(8).lipschitz if be == "rbpg" else d.lipschitz()
        ref = OB.run(a, batch.pixels, lam.cpu().numpy(), be, seeds=seeds.cpu().numpy(), lips=lips, max_iters=500, tol=1e-6, num_blocks=8)
        it = r.iterations.cpu().numpy(); rit = np.array([x["iterations"] for x in ref])
        ff = r.objective_final.cpu().numpy(); rf = np.array([x["f_final"] for x in ref])
        print(f"cfg{cfg_id} {be}: iters equal {np.mean(it == rit):.4f}  max|dit| {np.abs(it - rit).max()}  F rel max {np.max(np.abs(ff - rf) / rf):.2e}", flush=True)
RUNS = [(2, 262144, "rbpg"), (2, 262144, "fista"), (3, 65536, "rbpg"), (3, 65536, "fista")]
if os.environ.get("RUNS"):
    RUNS = [(int(c), int(p), b) for c, p, b in (r.split(":") for r in os.environ["RUNS"].split(","))]
for cfg_id, P, be in RUNS:
    batch = make_config(cfg_id, num_pixels=P)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    seeds = d.derive_seeds(2018, P)
    cfg = tb.SolverConfig(max_iters=500, tol=1e-6, num_blocks=8, seed=2018)
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
    print(f"cfg{cfg_id} {be} P={P}: {ms:.1f} ms  {P / ms * 1e3 / 1e6:.3f} M px/s  {its * flop / ms / 1e9:.2f} TFLOP/s algorithmic  mean iters {its / P:.1f}", flush=True)
