mkdir -p gpurun_out/meas2
timeout 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_tc_tiled.py -x -q 2>&1 | tail -1
for b in fista rbpg; do timeout 300 python tools/tiled_probe.py $b 512 20 2>&1 | grep -v Warn | tail -1; done
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/meas2/$name.json 2> gpurun_out/meas2/$name.err; echo "$name rc=$?"; }
run cfg4_fista --config 4 --backend fista --pixels 2048 --steps 2 --warmup 3
run cfg4_rbpg --config 4 --backend rbpg --pixels 2048 --steps 2 --warmup 3
run cfg5_rbpg --config 5 --backend rbpg --steps 1 --warmup 3
run cfg5_fista --config 5 --backend fista --steps 1 --warmup 3
