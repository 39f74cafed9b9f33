OUT=gpurun_out/r2d
mkdir -p $OUT

BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 2 --warmup 1 --pixels 131072 --no-cpu-baseline > $OUT/bench_gloo2.json 2> $OUT/bench_gloo2.err; echo "bench2 rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --pixels 131072 --no-cpu-baseline > $OUT/bench_1.json 2> $OUT/bench_1.err; echo "bench1 rc=$?"
