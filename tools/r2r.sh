OUT=gpurun_out/r2r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_simulate.py -q > $OUT/pytest_sim.txt 2>&1; echo "pytest rc=$?"
timeout 900 python tools/mc_bench.py 2000 > $OUT/mc_bench.json 2> $OUT/mc_bench.err; echo "mc rc=$?"
