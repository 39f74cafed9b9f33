OUT=gpurun_out/r2a
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench rc=$?"
timeout 600 compute-sanitizer --tool memcheck --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitizer_memcheck_smoke.txt 2>&1; echo "memcheck rc=$?"
