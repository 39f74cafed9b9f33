OUT=gpurun_out/r3f; mkdir -p $OUT
for XT in 0 1; do
echo "== XT=$XT"
TB_FISTA_XT=$XT ONECFG=1 KERNELS=warp,solo RUNS="2:65536:fista,2:8192:fista,1:8192:fista,2:16384:ista" timeout 600 python tools/ft_check.py 2>&1 | grep "cfg\|FT_CHECK"
done > $OUT/xt.txt 2>&1
cat $OUT/xt.txt
TB_FISTA_XT=1 KERNELS=warp,solo,team RUNS="1:1024:fista,1:37:ista,2:4099:fista" timeout 600 python tools/ft_check.py 2>&1 | grep "cfg\|FT_CHECK"
