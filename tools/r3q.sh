OUT=gpurun_out/r3q; mkdir -p $OUT
timeout 900 python bench.py --config 3 --backend rbpg --steps 2 --warmup 3 > $OUT/cfg3_rbpg.json 2> $OUT/cfg3_rbpg.err; echo "cfg3 rbpg rc=$?"
timeout 900 python bench.py --config 3 --backend fista --steps 2 --warmup 3 > $OUT/cfg3_fista.json 2> $OUT/cfg3_fista.err; echo "cfg3 fista rc=$?"
TB_WS_XTM=0 timeout 900 python bench.py --config 3 --backend rbpg --steps 2 --warmup 3 --no-cpu-baseline > $OUT/cfg3_rbpg_smemstate.json 2>/dev/null; echo "rc=$?"
TB_FISTA_KERNEL=warp timeout 900 python bench.py --config 3 --backend fista --steps 2 --warmup 3 --no-cpu-baseline > $OUT/cfg3_fista_warpkernel.json 2>/dev/null; echo "rc=$?"
for B in rbpg fista; do
  K=warp_solver; [ $B = fista ] && K=fista_tile
  CFG=3 P=32768 PREC=fp64 BACKEND=$B timeout 900 ncu --set full --clock-control none -k regex:$K -c 1 -f -o $OUT/n_$B python tools/prof_one.py > $OUT/n_$B.log 2>&1; echo "ncu $B rc=$?"
  ncu -i $OUT/n_$B.ncu-rep --page raw --csv > $OUT/n_$B.csv 2>/dev/null; rm -f $OUT/n_$B.ncu-rep
done
