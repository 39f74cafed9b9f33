OUT=gpurun_out/r3h; mkdir -p $OUT
CFG=2 P=65536 BACKEND=rbpg PREC=fp64 timeout 900 ncu --set full --import-source on --clock-control none -k regex:warp_solver -c 1 -f -o $OUT/rb python tools/prof_one.py > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/rb.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src.csv 2>/dev/null
ncu -i $OUT/rb.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
python tools/ncu_phases.py $OUT/src.csv paper_1805_01759_b200/csrc/k_warp_solver.cu 1 > $OUT/phases.txt 2>&1
python tools/ncu_top_lines.py $OUT/src.csv 45 > $OUT/top.txt 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r3h/src.csv')))
# opcode histogram weighted by executed count
import collections,re
hdr=None; h=collections.Counter()
for r in rows:
    if not r: continue
    if r[0]=='Line No': hdr=r; ii=hdr.index('Instructions Executed'); continue
    if hdr and r[0]=='' and len(r)>ii and r[2].startswith('0x'):
        op=r[3].strip().split()[0] if r[3].strip() else '?'
        if op.startswith('@'): op=r[3].strip().split()[1]
        op=op.split('.')[0]
        try: h[op]+=int(r[ii])
        except: pass
tot=sum(h.values())
open('gpurun_out/r3h/opcodes.txt','w').write('\n'.join(f'{k} {v} {100*v/tot:.1f}%' for k,v in h.most_common(40)))
PY
rm -f $OUT/rb.ncu-rep $OUT/src.csv
