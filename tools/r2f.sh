OUT=gpurun_out/r2f
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_c64.py -q -x > $OUT/pytest_c64.txt 2>&1; echo "pytest rc=$?"
CHK= RUNS=1:1024,2:262144,3:65536 timeout 900 python tools/c64_check.py > $OUT/timing.txt 2>&1; echo "timing rc=$?"
