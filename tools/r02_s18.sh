#!/bin/bash
# round 2, session 18: register-prefetched nrhs = 1 rows (row_accumulate_k1_pf)
# A/B vs the unprefetched rows and 3 CTAs/SM; bt_kernel two accumulator sets A/B;
# ncu full capture of the new nrhs = 1 kernel; GPU suite
cd $GRAFT_REPO_ROOT
O=gpurun_out/s18; mkdir -p $O
F=/tmp/cfg3.hvfm
ls -la $F > $O/cache.txt 2>&1
( time timeout 900 python -m pytest tests/test_gpu_parity.py -x -q ) > $O/pytest_parity.log 2>&1; echo "rc $?" >> $O/pytest_parity.log
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_pf.json 2> $O/bench_pf.err
for v in nopf pfc3; do VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err; done
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_pf.txt 2>&1
for k in 128 64; do
  timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k$k.json 2> $O/bench_k$k.err
  VF_LIB=paper_2209_07632_b200/build/var_acc2.so timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k${k}_acc2.json 2> $O/bench_k${k}_acc2.err
done
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_pf python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
echo done > $O/done
