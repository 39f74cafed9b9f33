"""Aggregate an ncu SASS source page by CUDA source line (needs the exact .so that was profiled).

usage: python tools/line_profile.py REPORT.ncu-rep LIB.so KERNEL_MANGLED_SUBSTR SOURCE.cu [units]
"""
import collections, csv, os, re, subprocess, sys, tempfile

rep, lib, kname, src = sys.argv[1:5]
units = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if os.path.basename(src).replace(".cu", "") in f]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin[0])], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(dis) if ".section" in l and ".text." in l and kname in l][0]
addr2line, cur = {}, None
for l in dis[start + 1:]:
    if ".section" in l and ".text." in l:
        break
    m = re.search(os.path.basename(src).replace(".", r"\.") + r'", line (\d+)', l)
    if m:
        cur = int(m.group(1))
    m2 = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m2 and cur is not None:
        addr2line[int(m2.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
ai, st, ie = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
addrs = [int(r[ai], 16) for r in data]
base = min(addrs)
by, bys = collections.Counter(), collections.Counter()
tot = tots = 0.0
for r, a in zip(data, addrs):
    ln = addr2line.get(a - base, -1)
    by[ln] += float(r[ie] or 0)
    bys[ln] += float(r[st] or 0)
    tot += float(r[ie] or 0)
    tots += float(r[st] or 0)
lines = open(src).read().split("\n")
print(f"total warp-instructions {tot:.4g}  ({tot / units:.1f} per unit)")
for ln, c in sorted(by.items(), key=lambda x: -x[1])[:40]:
    print(f"{ln:4d} {100 * c / tot:5.1f}% {c / units:7.1f}/u stall {100 * bys[ln] / tots:5.1f}%  {lines[ln - 1].strip()[:90] if ln > 0 else ''}")
