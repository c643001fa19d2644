#!/bin/bash
# round 2, session 32 (HEAD b0cddea + follow-ups): the evidence of r02_final.sh on
# the current build (GPU suite, smoke, default bench line, reference arm, ncu
# launch list, full captures of hot_kernel and bt_kernel), then the session-31
# A/Bs that never ran (phase-1 streamed V loads / x via L1, T rows via L1,
# FP32 resident batches DMMA vs FFMA)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s32; mkdir -p $O
F=/tmp/cfg3.hvfm
P=paper_2209_07632_b200
nvidia-smi > $O/nvidia_smi.txt 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
( time timeout 2400 python bench.py --fhat $F ) > $O/bench_default.json 2> $O/bench_default.err
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
for i in 1 2; do
  VF_LIB=$P/build/var_p1off.so timeout 600 $B > $O/bench_p1off_$i.json 2> $O/bench_p1off_$i.err
  VF_LIB=$P/build/var_p1na.so timeout 600 $B > $O/bench_p1na_$i.json 2> $O/bench_p1na_$i.err
  timeout 600 $B > $O/bench_p1new_$i.json 2> $O/bench_p1new_$i.err
  VF_LIB=$P/build/var_tl1.so timeout 600 $B > $O/bench_tl1_$i.json 2> $O/bench_tl1_$i.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 5 --warmup 3 > $O/ncu_launches.log 2>&1
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1 python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
timeout 300 python tools/mv_once.py 256 128 $F > $O/mv128_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_kernel -s 1 -c 1 -o $O/bt python tools/mv_once.py 256 128 $F > $O/ncu_bt.log 2>&1
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_k1.txt 2>&1
( time timeout 900 python bench.py --impl reference --steps 5 --warmup 3 ) > $O/bench_reference.json 2> $O/bench_reference.err
C="python bench.py --workload cfg2 --dtype f32 --no-cpu-baseline --steps 20"
for i in 1 2; do
  VF_LIB=$P/build/var_resffma.so timeout 600 $C > $O/bench_cfg2_f32_ffma_$i.json 2> $O/bench_cfg2_f32_ffma_$i.err
  timeout 600 $C > $O/bench_cfg2_f32_dmma_$i.json 2> $O/bench_cfg2_f32_dmma_$i.err
done
echo done > $O/done
