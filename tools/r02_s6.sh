#!/bin/bash
# round 2, session 6: bt v2, old k1 kernel with no-allocate loads, rows selftest
cd $GRAFT_REPO_ROOT
O=gpurun_out/s6; mkdir -p $O
F=/tmp/cfg3.hvfm
timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_rows.py tests/test_gpu_stream.py -x -q > $O/pytest_new.log 2>&1; echo "rc $?" >> $O/pytest_new.log
grep -q "rc 0" $O/pytest_new.log || exit 1
ls -la $F > $O/cache.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
timeout 900 python bench.py --fhat $F --no-cpu-baseline --steps 200 > $O/bench_default.json 2> $O/bench_default.err
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
VF_NO_STREAM=1 timeout 600 $B > $O/bench_old.json 2> $O/bench_old.err
VF_NO_STREAM=1 VF_LIB=paper_2209_07632_b200/build/var_na0.so timeout 600 $B > $O/bench_old_na0.json 2> $O/bench_old_na0.err
for k in 16 32 64 256; do
  timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k$k.json 2> $O/bench_k$k.err
done
for v in bts3 bts6; do
  VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs 128 --batched 0 --steps 10 > $O/bench_k128_$v.json 2> $O/bench_k128_$v.err
done
VF_NO_STREAM=1 timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
VF_NO_STREAM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1 python tools/mv_once.py 256 1 $F > $O/ncu.log 2>&1
echo done > $O/done
