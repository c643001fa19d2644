#!/bin/bash
# round 2, session 4: stream kernel v3 (bitmap piece lookup), variants; new GPU tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4; mkdir -p $O
F=/tmp/cfg3.hvfm
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > $O/pytest_stream.log 2>&1; echo "rc $?" >> $O/pytest_stream.log
grep -q "rc 0" $O/pytest_stream.log || exit 1
ls -la $F > $O/cache.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_default.json 2> $O/bench_default.err
for v in u4 u12 w16s2 w12s4; do
  VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err
done
timeout 900 python -m pytest tests/test_gpu_octree.py tests/test_gpu_timestep.py -q > $O/pytest_new.log 2>&1; echo "rc $?" >> $O/pytest_new.log
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_k1 -s 1 -c 1 -o $O/stream_k1 python tools/mv_once.py 256 1 $F > $O/ncu.log 2>&1
echo done > $O/done
