#!/bin/bash
# round 2, session 3: stream kernel v2 (two-pass consumer) tests, variants, ncu
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3; mkdir -p $O
F=/tmp/cfg3.hvfm
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > $O/pytest_stream.log 2>&1; echo "rc $?" >> $O/pytest_stream.log
grep -q "rc 0" $O/pytest_stream.log || exit 1
( time VF_LAYOUT_STATS=1 VF_BUILD_PROFILE=1 timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_default.json 2> $O/bench_default.err
for v in w12 w10s4 w16s2 u4 u16; do
  VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err
done
VF_NO_STREAM=1 timeout 600 $B > $O/bench_nostream.json 2> $O/bench_nostream.err
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_k1 -s 1 -c 1 -o $O/stream_k1 python tools/mv_once.py 256 1 $F > $O/ncu.log 2>&1
echo done > $O/done
