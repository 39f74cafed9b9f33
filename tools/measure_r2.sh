# Round-2 measurement sweep (GPU box): every config/backend bench line (with the reference CPU
# baselines), the reference arm, the default-bench launch list and a full ncu capture of the
# headline kernel.  Outputs in gpurun_out/meas_r2/.
OUT=gpurun_out/meas_r2
mkdir -p $OUT
nproc > $OUT/nproc.txt; lscpu | grep "Model name" >> $OUT/nproc.txt
run() { name=$1; shift; timeout 1500 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?"; }
run cfg2_rbpg_default
run ref_cfg2 --impl reference --steps 1 --warmup 1
run cfg2_fista --backend fista --steps 3 --warmup 3
run cfg1_rbpg --config 1 --backend rbpg --steps 5 --warmup 3
run cfg1_fista --config 1 --backend fista --steps 5 --warmup 3
run cfg3_rbpg --config 3 --backend rbpg --steps 2 --warmup 3
run cfg3_fista --config 3 --backend fista --steps 2 --warmup 3
run cfg4_rbpg_full --config 4 --backend rbpg --steps 1 --warmup 3
run cfg4_fista_full --config 4 --backend fista --steps 1 --warmup 3
run cfg5_rbpg --config 5 --backend rbpg --steps 1 --warmup 3
run cfg5_fista --config 5 --backend fista --steps 1 --warmup 3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_cfg2_rbpg_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:warp_solver -c 1 -o $OUT/ws_full -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --pixels 131072 > $OUT/ncu_full.log 2>&1; echo "full rc=$?"
