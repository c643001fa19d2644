#!/bin/bash
# round 2, session 28: bt_tc2_kernel variants (6 stage slots; cp.async producer)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s28; mkdir -p $O
F32=/tmp/cfg3_f32.hvfm
ls -la $F32 > $O/cache.txt 2>&1
for v in t2ldg t2s6 t2ldg6; do
  VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 python -m pytest tests/test_gpu_tiles.py -x -q > $O/pytest_tiles_$v.log 2>&1; echo "rc $?" >> $O/pytest_tiles_$v.log
done
B="python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --nrhs 128 --batched 0 --steps 10"
[ -f $F32 ] || timeout 2400 $B > $O/bench_build.json 2> $O/bench_build.err
VF_TC2=1 timeout 600 $B > $O/bench_tc2.json 2> $O/bench_tc2.err
for v in t2ldg t2s6 t2ldg6; do
  grep -q "rc 0" $O/pytest_tiles_$v.log && VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err
done
echo done > $O/done
