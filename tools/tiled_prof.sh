for b in rbpg fista; do timeout 300 python tools/cfg5_probe.py $b 20 2>&1 | grep -v Warn | tail -1; done
for b in rbpg fista; do timeout 300 python tools/tiled_probe.py $b 512 20 2>&1 | grep -v Warn | tail -1; done
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M --log-file gpurun_out/l_cfg5_rbpg.csv python tools/cfg5_probe.py rbpg 6 > /dev/null 2>&1; echo $?
timeout 600 ncu $M --log-file gpurun_out/l_cfg5_fista.csv python tools/cfg5_probe.py fista 6 > /dev/null 2>&1; echo $?
timeout 600 ncu $M --log-file gpurun_out/l_cfg4_rbpg.csv python tools/tiled_probe.py rbpg 512 6 > /dev/null 2>&1; echo $?
timeout 600 ncu $M --log-file gpurun_out/l_cfg4_fista.csv python tools/tiled_probe.py fista 512 6 > /dev/null 2>&1; echo $?
