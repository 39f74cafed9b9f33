OUT=gpurun_out/r3c; mkdir -p $OUT
TB_FISTA_KERNEL=${FK:-solo} CFG=${CFG:-2} P=${NP:-16384} BACKEND=fista PREC=fp64 timeout 900 ncu --set full --import-source on --clock-control none -k regex:fista_tile -c 1 -o $OUT/ft_full python tools/prof_one.py > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/ft_full.ncu-rep --page source --csv --print-source cuda,sass > $OUT/ft_source.csv 2>/dev/null
ncu -i $OUT/ft_full.ncu-rep --page raw --csv > $OUT/ft_raw.csv 2>/dev/null
ncu -i $OUT/ft_full.ncu-rep --page details > $OUT/ft_details.txt 2>/dev/null
python tools/ncu_phases.py $OUT/ft_source.csv paper_1805_01759_b200/csrc/k_fista_tile.cu 1 > $OUT/ft_phases.txt 2>&1
python tools/ncu_top_lines.py $OUT/ft_source.csv 50 > $OUT/ft_top.txt 2>&1
rm -f $OUT/ft_full.ncu-rep $OUT/ft_source.csv
