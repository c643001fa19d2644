#!/bin/bash
# round 2, session 7: row kernel with u16 offsets (default), bt with index prefetch
cd $GRAFT_REPO_ROOT
O=gpurun_out/s8; mkdir -p $O
F=/tmp/cfg3.hvfm
timeout 120 ./tools/tc_probe > $O/tc_probe.log 2>&1; echo "rc $?" >> $O/tc_probe.log
timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_stream.py tests/test_gpu_timestep.py -x -q > $O/pytest_new.log 2>&1; echo "rc $?" >> $O/pytest_new.log
grep -q "rc 0" $O/pytest_new.log || exit 1
ls -la $F > $O/cache.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
timeout 900 python bench.py --fhat $F --no-cpu-baseline --steps 200 > $O/bench_default.json 2> $O/bench_default.err
VF_K1_U32=1 timeout 600 python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200 > $O/bench_u32.json 2> $O/bench_u32.err
for k in 16 64 256; do
  timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k$k.json 2> $O/bench_k$k.err
done
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 300 python tools/mv_once.py 256 128 $F > $O/mv128_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_kernel -s 1 -c 1 -o $O/bt python tools/mv_once.py 256 128 $F > $O/ncu_bt.log 2>&1
echo done > $O/done
