# round-2 session 4: FISTA (cfg2) baseline for the CTA-tiled kernel: bench lines (warp, tiled path) and a source-level ncu capture
OUT=gpurun_out/r3a; mkdir -p $OUT
python bench.py --config 2 --backend fista --pixels 131072 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/cfg2_fista_warp.json 2> $OUT/cfg2_fista_warp.err; echo "warp rc=$?"
python bench.py --config 2 --backend fista --pixels 32768 --steps 1 --warmup 3 --no-cpu-baseline --path tiled > $OUT/cfg2_fista_tiled.json 2> $OUT/cfg2_fista_tiled.err; echo "tiled rc=$?"
python bench.py --config 3 --backend fista --pixels 32768 --steps 1 --warmup 3 --no-cpu-baseline --path tiled > $OUT/cfg3_fista_tiled.json 2> $OUT/cfg3_fista_tiled.err; echo "tiled3 rc=$?"
CFG=2 P=32768 BACKEND=fista PREC=fp64 timeout 900 ncu --set full --import-source on --clock-control none -k regex:warp_solver -c 1 -o $OUT/ws_fista_full python tools/prof_one.py > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/ws_fista_full.ncu-rep --page source --csv --print-source cuda,sass > $OUT/ws_fista_source.csv 2>/dev/null
ncu -i $OUT/ws_fista_full.ncu-rep --page raw --csv > $OUT/ws_fista_raw.csv 2>/dev/null
python tools/ncu_phases.py $OUT/ws_fista_source.csv paper_1805_01759_b200/csrc/k_warp_solver.cu 1 > $OUT/ws_fista_phases.txt 2>&1
ls -la $OUT
rm -f $OUT/ws_fista_full.ncu-rep
python - <<'PY'
import csv,sys
# keep only the per-line rows (cuda source lines), drop the SASS rows to keep the csv small
rows=list(csv.reader(open('gpurun_out/r3a/ws_fista_source.csv')))
w=csv.writer(open('gpurun_out/r3a/ws_fista_lines.csv','w'))
for r in rows:
    if r and (r[0] in('File Path','Line No') or r[0].isdigit()): w.writerow(r[:40])
PY
rm -f $OUT/ws_fista_source.csv
