# A/B of the tiled path (dev tool): bash tools/tiled_ab.sh lib1.so lib2.so ...
for L in "$@"; do
  echo "== $L"
  for cb in "4 fista --pixels 2048" "4 rbpg --pixels 2048" "5 fista" "5 rbpg"; do
    set -- $cb
    TB_LIB_PATH=$L timeout 600 python bench.py --config $1 --backend $2 ${3:-} ${4:-} --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg%s %s' % ('$1', '$2'), round(d['value'],2), 'px/s', round(d['ms_per_step'],1), 'ms/step frac', round(d['roofline']['frac'],3), 'iters', round(d['solver_stats']['mean_iterations'],1))"
  done
done
