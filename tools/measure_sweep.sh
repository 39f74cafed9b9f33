# Round measurement sweep (run on the GPU box): GPU tests, bench lines for every config/backend,
# the reference arm, the default-bench launch list and one full ncu capture of the headline kernel.
OUT=gpurun_out/meas
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1 > $OUT/pytest_gpu.txt
run() { name=$1; shift; timeout 900 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?"; }
run cfg2_rbpg_default
run cfg2_fista --backend fista --steps 3 --warmup 3
run cfg1_rbpg --config 1 --backend rbpg --steps 3 --warmup 3
run cfg1_fista --config 1 --backend fista --steps 3 --warmup 3
run cfg3_rbpg --config 3 --backend rbpg --steps 2 --warmup 3
run cfg3_fista --config 3 --backend fista --steps 2 --warmup 3
run cfg4_rbpg --config 4 --backend rbpg --pixels 2048 --steps 1 --warmup 3
run cfg4_fista --config 4 --backend fista --pixels 2048 --steps 1 --warmup 3
run cfg5_rbpg --config 5 --backend rbpg --steps 1 --warmup 3
run cfg5_fista --config 5 --backend fista --steps 1 --warmup 3
run ref_cfg2 --impl reference --steps 1 --warmup 3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_cfg2_rbpg_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:warp_solver -c 1 -o $OUT/ws_full \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --pixels 131072 > $OUT/ncu_full.log 2>&1; echo "full rc=$?"
