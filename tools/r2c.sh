OUT=gpurun_out/r2c
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_large_golden.py tests/test_gpu_parity.py -q -s -m gpu -k "large or own_lambda or cfg5 or cfg4" > $OUT/pytest_large.txt 2>&1; echo "pytest rc=$?"
