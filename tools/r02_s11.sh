#!/bin/bash
# round 2, session 11: k1 variants (no spill; wave mapping), FP32 cfg3 with tcgen05 tiles
cd $GRAFT_REPO_ROOT
O=gpurun_out/s11; mkdir -p $O
F=/tmp/cfg3.hvfm
F32=/tmp/cfg3_f32.hvfm
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_tiles.py -x -q > $O/pytest_new.log 2>&1; echo "rc $?" >> $O/pytest_new.log
grep -q "rc 0" $O/pytest_new.log || exit 1
ls -la $F $F32 > $O/cache.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_default.json 2> $O/bench_default.err
for v in wave wave8; do
  VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err
done
timeout 2400 python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --steps 100 > $O/bench_f32.json 2> $O/bench_f32.err
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1 python tools/mv_once.py 256 1 $F > $O/ncu.log 2>&1
echo done > $O/done
