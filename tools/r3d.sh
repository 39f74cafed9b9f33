OUT=gpurun_out/r3d; mkdir -p $OUT
for L in build/lib_scalar.so paper_1805_01759_b200/lib/libtomobpdn_b200.so build/lib_scalar.so paper_1805_01759_b200/lib/libtomobpdn_b200.so; do
  echo "== $L"
  for cb in "4 fista --pixels 2048" "5 fista"; do
    set -- $cb
    TB_LIB_PATH=$L timeout 600 python bench.py --config $1 --backend $2 ${3:-} ${4:-} --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg%s %s' % ('$1', '$2'), round(d['value'],2), 'px/s', round(d['ms_per_step'],1), 'ms/step frac', round(d['roofline']['frac'],3), 'iters', round(d['solver_stats']['mean_iterations'],1))"
  done
done > $OUT/tiled_ab.txt 2>&1
cat $OUT/tiled_ab.txt
