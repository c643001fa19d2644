#!/bin/bash
# round 2, session 23: bulk L2 prefetch of the nrhs = 1 row stream, A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s23; mkdir -p $O
F=/tmp/cfg3.hvfm
ls -la $F > $O/cache.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_base.json 2> $O/bench_base.err
for v in l2pf2 l2pf4 l2pf8; do VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err; done
timeout 600 $B > $O/bench_base2.json 2> $O/bench_base2.err
echo done > $O/done
