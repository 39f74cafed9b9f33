OUT=gpurun_out/r2g
mkdir -p $OUT
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --pixels 262144 > $OUT/cfg2.json 2>$OUT/cfg2.err; echo "cfg2 rc=$?"
timeout 600 python bench.py --config 3 --steps 2 --warmup 2 --no-cpu-baseline --pixels 65536 > $OUT/cfg3.json 2>$OUT/cfg3.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/cfg1.json 2>$OUT/cfg1.err; echo "cfg1 rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
