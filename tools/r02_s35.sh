#!/bin/bash
# round 2, session 35: transposed phase-1 reduction (VF_P1_TRED, default) vs the
# full butterfly (var_notred) on configs[2], then the round's last evidence on
# the default build: GPU suite, smoke, default bench line, ncu launch list, full
# capture of hot_kernel, phase trace, reference arm
cd $GRAFT_REPO_ROOT
O=gpurun_out/s35; mkdir -p $O
F=/tmp/cfg3.hvfm
P=paper_2209_07632_b200
nvidia-smi > $O/nvidia_smi.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
for i in 1 2 3; do
  VF_LIB=$P/build/var_notred.so timeout 600 $B > $O/bench_notred_$i.json 2> $O/bench_notred_$i.err
  timeout 600 $B > $O/bench_tred_$i.json 2> $O/bench_tred_$i.err
done
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_k1.txt 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
( time timeout 2400 python bench.py --fhat $F ) > $O/bench_default.json 2> $O/bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 5 --warmup 3 > $O/ncu_launches.log 2>&1
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1 python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
( time timeout 900 python bench.py --impl reference --steps 5 --warmup 3 ) > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --fhat $F --no-cpu-baseline --workload alg6 --steps 10 > $O/bench_alg6.json 2> $O/bench_alg6.err
timeout 900 python bench.py --fhat $F --workload cfg5 --steps 5 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
echo done > $O/done
