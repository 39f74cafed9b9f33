"""Top source lines of an ncu source-page csv by stall samples / instructions (dev tool).
    ncu -i REPORT --page source --csv --print-source cuda,sass > mixed.csv ; python tools/ncu_top_lines.py mixed.csv [N]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None; fname = None; cur = None
ins = collections.Counter(); st = collections.Counter(); text = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; ii = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None: continue
    if r[0] != "":
        if r[0].isdigit(): cur = (fname, int(r[0])); text[cur] = r[1][:110]
        continue
    if len(r) > max(ii, si) and r[2].startswith("0x") and cur:
        ins[cur] += int(r[ii]) if r[ii].isdigit() else 0
        st[cur] += int(r[si]) if r[si].isdigit() else 0
ti, ts = sum(ins.values()), sum(st.values())
print(f"total instr {ti} stall samples {ts}")
for key, v in st.most_common(N):
    print(f"{100.0 * v / max(ts,1):5.1f}% stall {100.0 * ins[key] / max(ti,1):5.1f}% instr  {key[0]}:{key[1]}  {text.get(key,'')}")
