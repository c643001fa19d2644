#!/bin/bash
# round 2, session 25: bt_tc_kernel with one A buffer pair and 2 CTAs per SM:
# parity (tiles tests through the variant library) and FP32 configs[2] nrhs = 128 A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s25; mkdir -p $O
F32=/tmp/cfg3_f32.hvfm
ls -la $F32 > $O/cache.txt 2>&1
VF_LIB=paper_2209_07632_b200/build/var_tcab1c2.so timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > $O/pytest_tiles_var.log 2>&1; echo "rc $?" >> $O/pytest_tiles_var.log
B="python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --nrhs 128 --batched 0 --steps 10"
timeout 2400 $B > $O/bench_f32_k128.json 2> $O/bench_f32_k128.err
VF_LIB=paper_2209_07632_b200/build/var_tcab1c2.so timeout 600 $B > $O/bench_f32_k128_tcab1c2.json 2> $O/bench_f32_k128_tcab1c2.err
VF_TC2=1 timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > $O/pytest_tiles_tc2.log 2>&1; echo "rc $?" >> $O/pytest_tiles_tc2.log
grep -q "rc 0" $O/pytest_tiles_tc2.log && VF_TC2=1 timeout 600 $B > $O/bench_f32_k128_tc2.json 2> $O/bench_f32_k128_tc2.err
echo done > $O/done
