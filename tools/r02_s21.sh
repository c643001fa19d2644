#!/bin/bash
# round 2, session 21: interleaved 16-bit CSR pieces (coalesced x gathers) A/B,
# parity of every nrhs = 1 path, column-split solve fix, ncu of the new kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/s21; mkdir -p $O
F=/tmp/cfg3.hvfm
ls -la $F > $O/cache.txt 2>&1
( time timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_k1p.py tests/test_gpu_timestep.py -x -q ) > $O/pytest_a.log 2>&1; echo "rc $?" >> $O/pytest_a.log
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_ilv.json 2> $O/bench_ilv.err
VF_K1_ILV=0 timeout 600 $B > $O/bench_plain.json 2> $O/bench_plain.err
VF_K1_OVL=1 timeout 600 $B > $O/bench_ilv_ovl.json 2> $O/bench_ilv_ovl.err
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace.txt 2>&1
timeout 1200 python tools/solve_cols.py $F 1,4,8 > $O/solve_cols.txt 2>&1
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
echo done > $O/done
