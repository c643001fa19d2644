#!/bin/bash
# round 2, session 31: nrhs = 1 phase 1 with streamed V loads (L1::no_allocate
# + L2 evict-first, VF_P1_NA) and x through L1 (VF_P1_L1) — A/B/C on
# configs[2] against variants built with the old loads; phase traces; the
# nrhs = 1 / ROWS GPU tests on the new build; T-row gathers through L1 (VF_K1_TL1);
# FP32 resident batches (configs[1] f32) on DMMA vs the FFMA loop
cd $GRAFT_REPO_ROOT
O=gpurun_out/s31; mkdir -p $O
F=/tmp/cfg3.hvfm
P=paper_2209_07632_b200
nvidia-smi > $O/nvidia_smi.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
for i in 1 2; do
  VF_LIB=$P/build/var_p1off.so timeout 600 $B > $O/bench_p1off_$i.json 2> $O/bench_p1off_$i.err
  VF_LIB=$P/build/var_p1na.so timeout 600 $B > $O/bench_p1na_$i.json 2> $O/bench_p1na_$i.err
  timeout 600 $B > $O/bench_p1new_$i.json 2> $O/bench_p1new_$i.err
  VF_LIB=$P/build/var_tl1.so timeout 600 $B > $O/bench_tl1_$i.json 2> $O/bench_tl1_$i.err
done
VF_LIB=$P/build/var_p1off.so timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_p1off.txt 2>&1
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_p1new.txt 2>&1
( time timeout 1500 python -m pytest tests/test_gpu_k1p.py tests/test_gpu_rows.py tests/test_gpu_parity.py -x -q ) > $O/pytest.log 2>&1; echo "rc $?" >> $O/pytest.log
C="python bench.py --workload cfg2 --dtype f32 --no-cpu-baseline --steps 20"
for i in 1 2; do
  VF_LIB=$P/build/var_resffma.so timeout 600 $C > $O/bench_cfg2_f32_ffma_$i.json 2> $O/bench_cfg2_f32_ffma_$i.err
  timeout 600 $C > $O/bench_cfg2_f32_dmma_$i.json 2> $O/bench_cfg2_f32_dmma_$i.err
done
echo done > $O/done
