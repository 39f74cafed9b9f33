OUT=gpurun_out/r3j; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; echo "gpu rc=$?"
tail -3 $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --config 3 --backend fista --steps 2 --warmup 3 > $OUT/cfg3_fista.json 2> $OUT/cfg3_fista.err; echo "cfg3 fista rc=$?"
timeout 900 python bench.py > $OUT/cfg2_rbpg_default.json 2> $OUT/default.err; echo "default rc=$?"
