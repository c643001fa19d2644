#!/bin/bash
# Dev tool (GPU box): final cfg3 evidence -- FP32 factors lines, FP64 nrhs=1 / 128
# lines with CPU baseline and parity, ncu launch list and full capture.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-cfg3final}
mkdir -p $O
timeout 1300 python bench.py --workload cfg3 --dtype f32 --nrhs 1 --steps 300 --warmup 5 --fhat /tmp/cfg3_f32.hvfm --no-cpu-baseline > $O/bench_cfg3_k1_f32.log 2>&1
timeout 300 python bench.py --workload cfg3 --dtype f32 --nrhs 128 --steps 10 --warmup 3 --fhat /tmp/cfg3_f32.hvfm --no-cpu-baseline --no-parity > $O/bench_cfg3_k128_f32.log 2>&1
timeout 1300 python tools/build_time.py 256 --save /tmp/cfg3_256.hvfm > $O/build_cfg3.log 2>&1
F=/tmp/cfg3_256.hvfm
timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --fhat $F > $O/bench_cfg3_k1.log 2>&1
timeout 300 python bench.py --workload cfg3 --nrhs 128 --steps 10 --warmup 3 --fhat $F --no-cpu-baseline > $O/bench_cfg3_k128.log 2>&1
timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 --fhat $F > $O/bench_cfg5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/ncu_launches_cfg3_k1.csv python bench.py --workload cfg3 --nrhs 1 --steps 3 --warmup 3 --fhat $F --no-cpu-baseline --no-parity > $O/ncu_launch_cfg3.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 3 -c 1 -o $O/hot_full_cfg3_k1 python tools/mv_once.py 256 1 $F > $O/ncu_full_cfg3.log 2>&1
echo done > $O/done
