#!/bin/bash
# round 2, session 20: nrhs = 1 row kernel without the phase barrier (item
# counter) + 3-row descriptor pipelining: parity, cfg3 A/B, trace, ncu
cd $GRAFT_REPO_ROOT
O=gpurun_out/s20; mkdir -p $O
F=/tmp/cfg3.hvfm
ls -la $F > $O/cache.txt 2>&1
( time timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k1 or matvec_same_blocks or column_split" ) > $O/pytest_k1.log 2>&1; echo "rc $?" >> $O/pytest_k1.log
( time timeout 900 python -m pytest tests/test_gpu_k1p.py tests/test_gpu_stream.py -x -q ) > $O/pytest_k1p.log 2>&1; echo "rc $?" >> $O/pytest_k1p.log
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_default.json 2> $O/bench_default.err
for v in noovl norowpf plainpf; do VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err; done
timeout 600 $B > $O/bench_default2.json 2> $O/bench_default2.err
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace.txt 2>&1
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
echo done > $O/done
