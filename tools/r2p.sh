OUT=gpurun_out/r2p; mkdir -p $OUT
CFG=2 P=32768 BACKEND=fista timeout 900 ncu --set full --import-source on --clock-control none -k regex:warp_solver -c 1 -o /tmp/ws_fista -f python tools/prof_one.py > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/ws_fista.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i /tmp/ws_fista.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src.csv 2>/dev/null
ls -la $OUT
