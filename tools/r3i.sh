for W in 13 12 11 10 9 8 6; do echo "TB_WARPS_L1=$W"; TB_WARPS_L1=$W RUNS="3:65536:rbpg" timeout 300 python tools/ab_solve.py 2>&1 | grep cfg; done
