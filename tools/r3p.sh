OUT=gpurun_out/r3p; mkdir -p $OUT
RUNS=3:65536 XW=16 timeout 600 python tools/xtm_check.py 2>&1 | grep "cfg\|XTM"
ONECFG=1 KERNELS=warp,solo RUNS="3:32768:fista,3:1501:ista" timeout 600 python tools/ft_check.py 2>&1 | grep "cfg\|FT_"
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; echo "gpu rc=$?"; tail -2 $OUT/pytest_gpu.txt
