# ncu --set full of the cfg3 instantiations (dictionary read through L1/L2): RBPG with the state in tensor
# memory / in shared memory, FISTA on the tensor-memory kernel / the warp kernel.  Raw metric pages only.
OUT=gpurun_out/r3n; mkdir -p $OUT
cap() { name=$1; kreg=$2; shift 2; env "$@" CFG=3 P=32768 PREC=fp64 timeout 900 ncu --set full --clock-control none -k regex:$kreg -c 1 -f -o $OUT/$name python tools/prof_one.py > $OUT/$name.log 2>&1; echo "$name rc=$?"; ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/$name.csv 2>/dev/null; rm -f $OUT/$name.ncu-rep; }
cap rbpg_tmem warp_solver BACKEND=rbpg
cap rbpg_smem warp_solver BACKEND=rbpg TB_WS_XTM=0
cap fista_tmem fista_tile BACKEND=fista
cap fista_warp warp_solver BACKEND=fista TB_FISTA_KERNEL=warp
