# Round-2 (session 4) measurement sweep on the GPU box: the FISTA lines on the tensor-memory kernel,
# the headline line again (unchanged kernel), the launch list of a cfg2 FISTA bench run and the
# ncu summaries of the three FISTA kernels.  Outputs in gpurun_out/meas_r2b/.
OUT=gpurun_out/meas_r2b
mkdir -p $OUT
run() { name=$1; shift; timeout 1500 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?"; }
run cfg2_rbpg_default
run cfg2_fista --backend fista --steps 3 --warmup 3
run cfg2_ista --backend ista --steps 2 --warmup 3 --pixels 262144
run cfg1_fista --config 1 --backend fista --steps 5 --warmup 3
run cfg3_fista --config 3 --backend fista --steps 2 --warmup 3
TB_FISTA_KERNEL=warp timeout 600 python bench.py --backend fista --steps 2 --warmup 3 --no-cpu-baseline > $OUT/cfg2_fista_warpkernel.json 2>/dev/null; echo "warp rc=$?"
TB_FISTA_KERNEL=team timeout 600 python bench.py --backend fista --steps 2 --warmup 3 --no-cpu-baseline > $OUT/cfg2_fista_teamkernel.json 2>/dev/null; echo "team rc=$?"
TB_FISTA_KERNEL=warp timeout 600 python bench.py --config 3 --backend fista --steps 2 --warmup 3 --no-cpu-baseline > $OUT/cfg3_fista_warpkernel.json 2>/dev/null; echo "warp3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_cfg2_fista.csv python bench.py --backend fista --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
for FK in solo team warp; do
  KREG=fista_tile; [ $FK = warp ] && KREG=warp_solver
  TB_FISTA_KERNEL=$FK CFG=2 P=32768 BACKEND=fista PREC=fp64 timeout 900 ncu --set full --import-source on --clock-control none -k regex:$KREG -c 1 -f -o $OUT/f_$FK python tools/prof_one.py > $OUT/ncu_$FK.log 2>&1; echo "ncu $FK rc=$?"
  ncu -i $OUT/f_$FK.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_$FK.csv 2>/dev/null
  ncu -i $OUT/f_$FK.ncu-rep --page raw --csv > $OUT/raw_$FK.csv 2>/dev/null
  SRC=paper_1805_01759_b200/csrc/k_fista_tile.cu; [ $FK = warp ] && SRC=paper_1805_01759_b200/csrc/k_warp_solver.cu
  python tools/ncu_phases.py $OUT/src_$FK.csv $SRC 1 > $OUT/phases_$FK.txt 2>&1
  python tools/ncu_top_lines.py $OUT/src_$FK.csv 30 > $OUT/top_$FK.txt 2>&1
  rm -f $OUT/f_$FK.ncu-rep $OUT/src_$FK.csv
done
