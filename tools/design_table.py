"""Regenerate the DESIGN.md §8 measurement table from profiles/r1_measurements/*.json (dev tool)."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = os.path.join(ROOT, "profiles", "r1_measurements")

ROWS = [
    ("cfg1_rbpg", "cfg1 (1,024 px, n=25, m=200)", "RBPG"),
    ("cfg1_fista", "cfg1", "FISTA"),
    ("cfg2_rbpg_default", "**cfg2 (1,048,576 px, n=25, m=300)**", "**RBPG**"),
    ("cfg2_fista", "cfg2", "FISTA"),
    ("cfg3_rbpg", "cfg3 (262,144 px, n=50, m=512)", "RBPG"),
    ("cfg3_fista", "cfg3", "FISTA"),
    ("cfg4_rbpg_full", "cfg4 (full 16,384 px, m=160,000)", "RBPG"),
    ("cfg4_rbpg", "cfg4 (2,048-px subset)", "RBPG"),
    ("cfg4_fista_full", "cfg4 (full 16,384 px)", "FISTA"),
    ("cfg4_fista", "cfg4 (2,048-px subset)", "FISTA"),
    ("cfg5_fista", "cfg5 (64 RHS, m=1,048,576, 1 GPU)", "FISTA"),
    ("cfg5_rbpg", "cfg5", "RBPG"),
]


def big(x):
    e = len(str(int(x))) - 1
    return f"≈{x / 10 ** e:.1f}×10^{e}×"


def px(v):
    return f"{v / 1e6:.2f} M" if v >= 1e5 else (f"{v:,.0f}" if v >= 100 else f"{v:.1f}")


def main():
    out = ["| workload | backend | px/s device | e2e px/s | FP32 roofline | launches/step | CPU px/s (16 cores) | e2e speed-up |",
           "|---|---|---|---|---|---|---|---|"]
    for name, wl, be in ROWS:
        d = json.load(open(os.path.join(M, name + ".json")))
        c = d.get("cpu_baseline") or {}
        e2e = (d.get("e2e") or {}).get("value", 0.0)
        frac = 100 * d["roofline"]["frac"]
        steps = d.get("steps") or 1
        launches = d.get("gpu_launches")
        lps = f"{launches // steps:,}" if launches else "—"
        if c.get("value"):
            cpu = f"{c['value']:,.0f}" if c["value"] >= 10 else f"{c['value']:.2g}"
            sp = e2e / c["value"]
            spd = f"{sp:,.0f}×" if sp < 1e4 else big(sp)
        else:
            cpu, spd = ("≈8.5e-5 (SURVEY §0 estimate)", big(e2e / 8.5e-5)) if "fista" in name else ("—", "—")
        bold = name == "cfg2_rbpg_default"
        f = lambda s: f"**{s}**" if bold else s
        out.append(f"| {wl} | {be} | {f(px(d['value']))} | {f(px(e2e))} | {f(f'{frac:.1f}%')} | {f(lps)} | {f(cpu)} | {f(spd)} |")
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    i0 = s.index("| workload | backend | px/s device |")
    i1 = s.index("\n\n", i0)
    note = ("\n\ncfg4 CPU column: 10 fixed iterations per pixel (plus the reference's per-solve power "
            "iterations), rate scaled by the GPU's mean iteration count; cfg5 CPU: the SURVEY §0 per-RHS estimate.")
    s = s[:i0] + "\n".join(out) + note + s[i1:]
    open(p, "w").write(s)
    print("\n".join(out))


if __name__ == "__main__":
    main()
