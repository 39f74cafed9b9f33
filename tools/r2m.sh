OUT=gpurun_out/r2m; mkdir -p $OUT
M="--metrics gpu__time_duration.sum --clock-control none --csv"
CFG=5 BACKEND=rbpg ITERS=20 timeout 600 ncu $M --log-file $OUT/l_cfg5_rbpg.csv python tools/tiled_rounds.py > /dev/null 2>&1; echo $?
CFG=5 BACKEND=fista ITERS=10 timeout 600 ncu $M --log-file $OUT/l_cfg5_fista.csv python tools/tiled_rounds.py > /dev/null 2>&1; echo $?
CFG=4 P=2048 BACKEND=rbpg ITERS=20 timeout 600 ncu $M --log-file $OUT/l_cfg4_rbpg.csv python tools/tiled_rounds.py > /dev/null 2>&1; echo $?
