OUT=gpurun_out/r2b
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --backend fista --steps 3 --warmup 3 --no-cpu-baseline > $OUT/cfg2_fista.json 2> $OUT/cfg2_fista.err; echo "fista rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/cfg2_rbpg.json 2> $OUT/cfg2_rbpg.err; echo "rbpg rc=$?"
