OUT=gpurun_out/r2n; mkdir -p $OUT
CFG=5 BACKEND=rbpg ITERS=40 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tiled_pass -s 30 -c 1 -o $OUT/pass_cfg5_rbpg -f python tools/tiled_rounds.py > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
