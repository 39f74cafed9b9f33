mkdir -p gpurun_out/meas
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1 > gpurun_out/meas/pytest_gpu.txt
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/meas/$name.json 2> gpurun_out/meas/$name.err; echo "$name rc=$?"; }
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
