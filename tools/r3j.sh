# final check of HEAD on the GPU box: the full GPU test suite, smoke(), the default bench line and the reference arm
OUT=gpurun_out/r3j; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; echo "gpu rc=$?"
tail -3 $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/cfg2_rbpg_default.json 2> $OUT/default.err; echo "default rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $OUT/ref_cfg2.json 2> $OUT/ref.err; echo "ref rc=$?"
