OUT=gpurun_out/r2j; mkdir -p $OUT
python tools/ab_solve.py > $OUT/ab.txt 2>&1
for c in "2 65536" "3 32768" "1 1024"; do set -- $c
  timeout 900 python bench.py --config $1 --backend fista --path tiled --pixels $2 --steps 2 --warmup 2 --no-cpu-baseline > $OUT/tiled_fista_cfg$1.json 2>$OUT/tiled_fista_cfg$1.err; echo "tiled cfg$1 rc=$?"
  timeout 900 python bench.py --config $1 --backend fista --pixels $2 --steps 2 --warmup 2 --no-cpu-baseline > $OUT/warp_fista_cfg$1.json 2>$OUT/warp_fista_cfg$1.err; echo "warp cfg$1 rc=$?"
done
