#!/bin/bash
# round 2, session 24: two rounds of the nrhs = 1 stream in registers (4 CTAs
# with spills / 3 CTAs), FP32 configs[2] line on the current kernels, Alg. 6 and
# cfg5 lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/s24; mkdir -p $O
F=/tmp/cfg3.hvfm
F32=/tmp/cfg3_f32.hvfm
ls -la $F $F32 > $O/cache.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_base.json 2> $O/bench_base.err
for v in pfd2c4 pfd2c3; do VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err; done
timeout 600 $B > $O/bench_base2.json 2> $O/bench_base2.err
timeout 900 python bench.py --fhat $F --no-cpu-baseline --workload alg6 --steps 10 > $O/bench_alg6.json 2> $O/bench_alg6.err
timeout 900 python bench.py --fhat $F --workload cfg5 --steps 5 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
( time timeout 2400 python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --steps 100 ) > $O/bench_f32.json 2> $O/bench_f32.err
echo done > $O/done
