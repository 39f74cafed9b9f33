for i in 1 2 3; do timeout 300 python bench.py --config 5 --backend rbpg --steps 1 --warmup 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench rbpg', round(d['value'],2), round(d['ms_per_step'],1))"; done
for i in 1 2; do timeout 300 python tools/cfg5_probe.py rbpg 500 2>&1 | grep -v Warn | tail -1; done
