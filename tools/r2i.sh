OUT=gpurun_out/r2i; mkdir -p $OUT
python tools/ab_solve.py > $OUT/ab.txt 2>&1
TB_LIB_PATH=build/lib_noshfl.so python tools/ab_solve.py >> $OUT/ab.txt 2>&1
python tools/ab_solve.py >> $OUT/ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"
