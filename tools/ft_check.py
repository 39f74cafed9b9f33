"""Team-tiled FISTA/ISTA kernel vs the warp-per-pixel kernel (GPU dev tool): byte identity of every output and timings.

RUNS="cfg:pixels:backend,..."  (default: cfg1/cfg2 FISTA + ISTA, odd batch sizes)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config

RUNS = [(int(c), int(p), b) for c, p, b in (x.split(":") for x in os.environ.get(
    "RUNS", "1:1024:fista,1:37:fista,1:1:fista,1:1024:ista,2:8192:fista,2:4099:ista,2:65536:fista").split(",") if x)]
CFGS = [dict(max_iters=500, tol=1e-6), dict(max_iters=120, tol=1e-6, alpha_init_scale=4.0), dict(max_iters=40, tol=1e-6, fixed_iters=40)]
KERNELS = os.environ.get("KERNELS", "warp,team,solo").split(",")
bad = 0
for cfg_id, P, be in RUNS:
    batch = make_config(cfg_id, num_pixels=P)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    for ci, kw in enumerate(CFGS if (P <= 8192 and not os.environ.get("ONECFG")) else CFGS[:1]):
        cfg = tb.SolverConfig(num_blocks=8, **kw)
        res = {}
        for kern in KERNELS:
            os.environ["TB_FISTA_KERNEL"] = kern
            hist = P <= 8192
            r = d.solve(px, lam, cfg, be, history=hist)
            torch.cuda.synchronize()
            ts = []
            for _ in range(2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); r = d.solve(px, lam, cfg, be, history=hist); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[kern] = (r, min(ts))
        rw, rt = res[KERNELS[0]][0], res[KERNELS[-1]][0]
        same = {
            "x": torch.equal(rw.x_hat.view(torch.int64), rt.x_hat.view(torch.int64)),
            "F": torch.equal(rw.objective_final.view(torch.int64), rt.objective_final.view(torch.int64)),
            "it": torch.equal(rw.iterations, rt.iterations),
            "st": torch.equal(rw.status, rt.status),
        }
        if rw.history is not None:
            same["hist"] = torch.equal(torch.nan_to_num(rw.history, nan=-1.0), torch.nan_to_num(rt.history, nan=-1.0))
        okay = all(same.values())
        bad += not okay
        its = rt.iterations.double().sum().item()
        flop = 16.0 * batch.n * batch.m
        extra = ""
        if not okay:
            nd = (rw.iterations != rt.iterations).sum().item()
            fx = (rw.objective_final - rt.objective_final).abs().max().item()
            extra = f" iter-diff pixels {nd}, max |dF| {fx:.3e}, it warp/tile {rw.iterations[:6].tolist()} {rt.iterations[:6].tolist()}"
        print(f"cfg{cfg_id} {be} P={P} cfg#{ci}: identical={okay} {same if not okay else ''}{extra} | {' '.join(f'{k} {res[k][1]:.2f} ms' for k in KERNELS)} "
              f"({res[KERNELS[0]][1] / res[KERNELS[-1]][1]:.2f}x)  {KERNELS[-1]} {its * flop / res[KERNELS[-1]][1] / 1e9 / 70.78:.4f} of FP32, status counts {torch.bincount(rt.status, minlength=4).tolist()}", flush=True)
print("FT_CHECK", "FAIL" if bad else "OK")
sys.exit(1 if bad else 0)
