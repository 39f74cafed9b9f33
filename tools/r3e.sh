OUT=gpurun_out/r3e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fista_tmem.py -q -x > $OUT/pytest_tmem.txt 2>&1; echo "tmem rc=$?"
tail -4 $OUT/pytest_tmem.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; echo "gpu rc=$?"
tail -4 $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"
