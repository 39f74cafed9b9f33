"""Per-phase instruction/stall breakdown of an ncu source capture (dev tool).

    ncu -i REPORT --page source --csv --print-source cuda,sass > mixed.csv
    python tools/ncu_phases.py mixed.csv SOURCE.cu UNITS

Phases are the "// ---- " comment markers of SOURCE.cu (a marker opens a phase that lasts until
the next one); device helpers above the kernel are their own phases; lines of other files are
grouped per file (common.cuh is the FFMA2 asm of the adjoint).  UNITS normalises the counts
(e.g. pixel-iterations in the captured launch)."""
import collections
import csv
import re
import sys


def phases_of(src):
    lines = open(src).read().splitlines()
    names, cur = {}, "prologue"
    for i, l in enumerate(lines, 1):
        m = re.match(r"\s*// ---- (.*)", l)
        if m:
            cur = m.group(1).split("(")[0].strip()[:40]
        elif re.match(r"(template|__global__|__device__|auto forward_list)", l.strip()):
            mm = re.search(r"(\w+)\s*\(", l.strip().replace("__launch_bounds__", ""))
            if "forward_list" in l:
                cur = "forward_list (sparse fp64 A z)"
            elif l.strip().startswith("__global__") or l.strip().startswith("__device__"):
                cur = "helper " + (mm.group(1) if mm else "?")
        names[i] = cur
        if l.strip() == "};" and cur.startswith("forward_list"):
            cur = "kernel body"
    return names


def main():
    path, src, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
    base = src.split("/")[-1]
    ph = phases_of(src)
    rows = list(csv.reader(open(path)))
    hdr = cur = fname = None
    ins, st = collections.Counter(), collections.Counter()
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None:
            continue
        if r[0] != "":
            if r[0].isdigit():
                cur = (fname, int(r[0]))
            continue
        if len(r) > ii and r[2].startswith("0x") and cur:
            key = ph.get(cur[1], "?") if cur[0] == base else "file " + cur[0]
            ins[key] += int(r[ii]) if r[ii].isdigit() else 0
            st[key] += int(r[si]) if r[si].isdigit() else 0
    ti, ts = sum(ins.values()), max(sum(st.values()), 1)
    print(f"| phase | warp-instr per unit | share | stall-sample share |\n|---|---|---|---|")
    for k, v in ins.most_common():
        print(f"| {k} | {v / units:.1f} | {100 * v / ti:.1f}% | {100 * st[k] / ts:.1f}% |")
    print(f"| **total** | **{ti / units:.1f}** | | |")


if __name__ == "__main__":
    main()
