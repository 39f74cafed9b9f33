#!/bin/bash
# Build A/B variants of the warp solver library into build/ (dev tool): each VAR="NAME:-DFLAGS"
set -e
cd "$(dirname "$0")/.."
C=paper_1805_01759_b200/csrc
ARCH="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
mkdir -p build/objs
for f in tb_api k_setup k_select k_tiled k_tc_tiled; do
  if [ ! -f build/objs/$f.o ] || [ $C/$f.cu -nt build/objs/$f.o ]; then nvcc $ARCH -c $C/$f.cu -o build/objs/$f.o & fi
done
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  nvcc $ARCH $flags -c $C/k_warp_solver.cu -o build/objs/ws_$name.o &
done
wait
for v in "$@"; do
  name=${v%%:*}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/lib_$name.so build/objs/ws_$name.o build/objs/tb_api.o build/objs/k_setup.o build/objs/k_select.o build/objs/k_tiled.o build/objs/k_tc_tiled.o
done
ls -la build/*.so
