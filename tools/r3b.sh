OUT=gpurun_out/r3b; mkdir -p $OUT
timeout 300 python tools/ft_check.py > $OUT/ft_check.txt 2>&1; echo "ft_check rc=$?"
tail -30 $OUT/ft_check.txt
