OUT=gpurun_out/r2q; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_edges.py -q > $OUT/pytest_edges.txt 2>&1; echo "edges rc=$?"
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.txt 2>&1; echo "gpu rc=$?"
