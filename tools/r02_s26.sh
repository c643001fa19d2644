#!/bin/bash
# round 2, session 26: tc2 with the flattened producer (index prefetch), FP32
# nrhs = 128 A/B; ROWS iterations on the 16-bit layout (rows tests + cfg5 line)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s26; mkdir -p $O
F=/tmp/cfg3.hvfm
F32=/tmp/cfg3_f32.hvfm
ls -la $F $F32 > $O/cache.txt 2>&1
VF_TC2=1 timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > $O/pytest_tiles_tc2.log 2>&1; echo "rc $?" >> $O/pytest_tiles_tc2.log
( time timeout 900 python -m pytest tests/test_gpu_rows.py -x -q ) > $O/pytest_rows.log 2>&1; echo "rc $?" >> $O/pytest_rows.log
if [ -f $F32 ]; then
  B="python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --nrhs 128 --batched 0 --steps 10"
  grep -q "rc 0" $O/pytest_tiles_tc2.log && VF_TC2=1 timeout 600 $B > $O/bench_f32_k128_tc2.json 2> $O/bench_f32_k128_tc2.err
  timeout 600 $B > $O/bench_f32_k128.json 2> $O/bench_f32_k128.err
fi
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
grep -q "rc 0" $O/pytest_rows.log && timeout 900 python bench.py --fhat $F --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200 > $O/bench_default.json 2> $O/bench_default.err
echo done > $O/done
