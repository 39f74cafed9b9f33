# ncu --set full of one late tiled_pass_kernel launch (cfg4 FISTA, 2,048 px) with source-level hot lines
OUT=gpurun_out/r3r; mkdir -p $OUT
TB_TILED_GRAPH=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tiled_pass -s 300 -c 1 -f -o $OUT/tp python bench.py --config 4 --backend fista --pixels 2048 --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/tp.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src.csv 2>/dev/null
ncu -i $OUT/tp.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
python tools/ncu_top_lines.py $OUT/src.csv 40 > $OUT/top.txt 2>&1
rm -f $OUT/tp.ncu-rep $OUT/src.csv
