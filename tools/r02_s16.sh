#!/bin/bash
# round 2, session 16: phase trace of the nrhs = 1 row kernel on configs[2],
# bt_kernel zero-fragment skip A/B at nrhs = 16/64/128, the GPU suite minus the
# flags test, compute-sanitizer racecheck of the small all-kernels case
cd $GRAFT_REPO_ROOT
O=gpurun_out/s16; mkdir -p $O
F=/tmp/cfg3.hvfm
ls -la $F > $O/cache.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_k1.txt 2>&1
for k in 128 64 16; do
  timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k$k.json 2> $O/bench_k$k.err
  VF_LIB=paper_2209_07632_b200/build/var_noskip.so timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k${k}_noskip.json 2> $O/bench_k${k}_noskip.err
done
( time timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_gpu_parity.py::test_k1_matvec_flags_equal_barrier_bitwise ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 600 python tools/sanitize_case.py > $O/san_plain.log 2>&1; echo "rc $?" >> $O/san_plain.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_case.py > $O/racecheck.log 2>&1; echo "rc $?" >> $O/racecheck.log
echo done > $O/done
