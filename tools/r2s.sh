OUT=gpurun_out/r2s; mkdir -p $OUT
python tools/ab_solve.py > $OUT/ab.txt 2>&1
python tools/ab_solve.py >> $OUT/ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"
