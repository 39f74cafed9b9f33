"""RBPG warp kernel with the dictionary read through L1 (cfg3): x in tensor memory (XTM) vs x in shared
memory (GPU dev tool).  Byte identity of every output and timings; RUNS="cfg:pixels,...", XW = warp caps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_01759_b200 as tb
from paper_1805_01759_b200.synth import make_config

RUNS = [(int(c), int(p)) for c, p in (x.split(":") for x in os.environ.get("RUNS", "3:4096,3:65536").split(","))]
XW = [int(x) for x in os.environ.get("XW", "16,14,12").split(",")]
bad = 0
for cfg_id, P in RUNS:
    batch = make_config(cfg_id, num_pixels=P)
    d = tb.Dictionary(batch.dictionary)
    px = torch.from_numpy(batch.pixels).cuda()
    lam = d.default_lambda(px, 0.1)
    seeds = d.derive_seeds(2018, P)
    for kw in (dict(max_iters=500, tol=1e-6), dict(max_iters=60, tol=1e-6, alpha_init_scale=4.0)):
        cfg = tb.SolverConfig(num_blocks=8, seed=2018, **kw)
        res = {}
        for name, env in [("smem", {"TB_WS_XTM": "0"})] + [(f"xtm{w}", {"TB_WS_XTM": "1", "TB_WARPS_CAP": str(w)}) for w in XW]:
            for k in ("TB_WS_XTM", "TB_WARPS_CAP"):
                os.environ.pop(k, None)
            os.environ.update(env)
            hist = P <= 8192
            r = d.solve(px, lam, cfg, "rbpg", seeds=seeds, history=hist)
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); r = d.solve(px, lam, cfg, "rbpg", seeds=seeds, history=hist); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[name] = (r, min(ts))
        ref = res["smem"][0]
        line = f"cfg{cfg_id} P={P} {kw.get('alpha_init_scale', 1)}: smem {res['smem'][1]:.2f} ms"
        for name in list(res)[1:]:
            r = res[name][0]
            same = (torch.equal(r.x_hat.view(torch.int64), ref.x_hat.view(torch.int64)) and torch.equal(r.objective_final.view(torch.int64), ref.objective_final.view(torch.int64))
                    and torch.equal(r.iterations, ref.iterations) and torch.equal(r.status, ref.status)
                    and (ref.history is None or torch.equal(torch.nan_to_num(r.history, nan=-1.0), torch.nan_to_num(ref.history, nan=-1.0))))
            bad += not same
            line += f" | {name} {res[name][1]:.2f} ms ({res['smem'][1] / res[name][1]:.3f}x) identical={same}"
        print(line, flush=True)
print("XTM_CHECK", "FAIL" if bad else "OK")
