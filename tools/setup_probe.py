"""Setup-kernel probe (GPU): default_lambda and power-iteration timings per config (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config, lambda_from_beta

for cfg_id, P in ((2, 1 << 20), (4, 2048), (5, 64)):
    batch = make_config(cfg_id, num_pixels=P)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        lam = d.default_lambda(px, 0.1)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    sub = min(P, 256)
    ref = lambda_from_beta(batch.dictionary, batch.pixels[:sub], 0.1)
    rel = float(np.max(np.abs(lam[:sub].cpu().numpy() - ref) / ref))
    flop = 8.0 * batch.n * batch.m * P
    print(f"cfg{cfg_id} default_lambda P={P}: {ms:.3f} ms  {flop / ms / 1e9:.1f} TFLOP/s  max rel vs fp64 host {rel:.2e}", flush=True)
    if cfg_id >= 4:
        t0 = time.time(); lf = d.lipschitz(); t1 = time.time(); part = d.partition(8); t2 = time.time()
        print(f"cfg{cfg_id} power iterations: full {1e3 * (t1 - t0):.1f} ms (L={lf:.6e}), 8 blocks {1e3 * (t2 - t1):.1f} ms", flush=True)
