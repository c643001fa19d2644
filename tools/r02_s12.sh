#!/bin/bash
# round 2, session 12: re-baseline after the container restore -- full GPU suite,
# smoke, the driver's default bench (builds configs[2] F-hat), reference arm,
# nrhs = 1 kernel variants, launch list + full capture of the hot kernel, FP32 line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s12; mkdir -p $O
F=/tmp/cfg3.hvfm
F32=/tmp/cfg3_f32.hvfm
nvidia-smi > $O/nvidia_smi.txt 2>&1
( time timeout 1800 python -m pytest tests -m gpu -x -q ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
ls -la $F $F32 > $O/cache.txt 2>&1
( time timeout 2400 python bench.py --fhat $F ) > $O/bench_default.json 2> $O/bench_default.err
( time timeout 900 python bench.py --impl reference --steps 5 --warmup 3 ) > $O/bench_reference.json 2> $O/bench_reference.err
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
VF_K1_KERNEL=stream timeout 600 $B > $O/bench_stream.json 2> $O/bench_stream.err
VF_LIB=paper_2209_07632_b200/build/var_wave.so timeout 600 $B > $O/bench_wave.json 2> $O/bench_wave.err
for k in 4 16 64; do
  timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k$k.json 2> $O/bench_k$k.err
done
timeout 900 python bench.py --fhat $F --no-cpu-baseline --workload alg6 --steps 10 > $O/bench_alg6.json 2> $O/bench_alg6.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 5 --warmup 3 > $O/ncu_launches.log 2>&1
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1 python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
timeout 300 python tools/mv_once.py 256 128 $F > $O/mv128_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_kernel -s 1 -c 1 -o $O/bt python tools/mv_once.py 256 128 $F > $O/ncu_bt.log 2>&1
( time timeout 2400 python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --steps 100 ) > $O/bench_f32.json 2> $O/bench_f32.err
echo done > $O/done
