OUT=gpurun_out/r3g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_select_adversarial.py -q > $OUT/pytest.txt 2>&1; echo "rc=$?"
grep -v Warning $OUT/pytest.txt | tail -40
