OUT=gpurun_out/r2l; mkdir -p $OUT
timeout 900 python tools/graph_ab.py > $OUT/graph_ab.txt 2>&1; echo "ab rc=$?"
timeout 1200 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_large_golden.py tests/test_gpu_multiproc.py -q -x > $OUT/pytest_tiled.txt 2>&1; echo "pytest rc=$?"
