#!/bin/bash
# round 2, session 34: shuffle-free round mapping (VF_K1_NOSHFL, default) vs the
# shuffle build (var_shfl), with T rows through L1 (default) and through L2 only, on configs[2], then the round's final evidence on the
# default build: GPU suite, smoke, default bench line, reference arm, ncu launch
# list, full capture of hot_kernel, phase trace
cd $GRAFT_REPO_ROOT
O=gpurun_out/s34; mkdir -p $O
F=/tmp/cfg3.hvfm
P=paper_2209_07632_b200
nvidia-smi > $O/nvidia_smi.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
for i in 1 2 3; do
  VF_LIB=$P/build/var_shfl.so timeout 600 $B > $O/bench_shfl_$i.json 2> $O/bench_shfl_$i.err
  timeout 600 $B > $O/bench_noshfl_$i.json 2> $O/bench_noshfl_$i.err
  VF_K1_TL1=0 timeout 600 $B > $O/bench_noshfl_tl0_$i.json 2> $O/bench_noshfl_tl0_$i.err
  VF_LIB=$P/build/var_shfl.so VF_K1_TL1=0 timeout 600 $B > $O/bench_shfl_tl0_$i.json 2> $O/bench_shfl_tl0_$i.err
done
( time timeout 1800 python -m pytest tests -m gpu -q ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
( time timeout 2400 python bench.py --fhat $F ) > $O/bench_default.json 2> $O/bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 5 --warmup 3 > $O/ncu_launches.log 2>&1
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1 python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_k1.txt 2>&1
( time timeout 900 python bench.py --impl reference --steps 5 --warmup 3 ) > $O/bench_reference.json 2> $O/bench_reference.err
( time timeout 1200 python bench.py --fhat /tmp/cfg3_f32.hvfm --dtype f32 --no-cpu-baseline --batched 0 --steps 100 ) > $O/bench_f32.json 2> $O/bench_f32.err
echo done > $O/done
