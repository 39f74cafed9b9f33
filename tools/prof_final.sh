OUT=gpurun_out/meas7; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_cfg2_rbpg_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:warp_solver -c 1 -o $OUT/ws_full \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --pixels 131072 > $OUT/ncu_full.log 2>&1; echo "full rc=$?"
