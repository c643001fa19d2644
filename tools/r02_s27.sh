#!/bin/bash
# round 2, session 27: ncu of the FP32 tcgen05 tile kernels (v1, warp-specialised v2)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s27; mkdir -p $O
F32=/tmp/cfg3_f32.hvfm
ls -la $F32 > $O/cache.txt 2>&1
[ -f $F32 ] || timeout 2400 python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --nrhs 128 --batched 0 --steps 3 > $O/bench_build.json 2> $O/bench_build.err
VF_TC2=1 timeout 300 python tools/mv_once.py 256 128 $F32 > $O/mv_tc2.log 2>&1 && \
VF_TC2=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_tc2 -s 1 -c 1 -o $O/tc2 python tools/mv_once.py 256 128 $F32 > $O/ncu_tc2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_tc_kernel -s 1 -c 1 -o $O/tc1 python tools/mv_once.py 256 128 $F32 > $O/ncu_tc1.log 2>&1
echo done > $O/done
