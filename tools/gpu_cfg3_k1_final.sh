#!/bin/bash
# Dev tool (GPU box): final cfg3 nrhs=1 evidence (bench with CPU baseline + parity,
# ncu launch list + full capture, phase trace), and the cfg5 line.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-cfg3k1}
mkdir -p $O
timeout 1300 python tools/build_time.py 256 --save /tmp/cfg3_256.hvfm > $O/build_cfg3.log 2>&1
F=/tmp/cfg3_256.hvfm
timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --fhat $F > $O/bench_cfg3_k1.log 2>&1
timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 --fhat $F > $O/bench_cfg5.log 2>&1
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_cfg3_k1.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/ncu_launches_cfg3_k1.csv python bench.py --workload cfg3 --nrhs 1 --steps 3 --warmup 3 --fhat $F --no-cpu-baseline --no-parity > $O/ncu_launch_cfg3.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 3 -c 1 -o $O/hot_full_cfg3_k1 python tools/mv_once.py 256 1 $F > $O/ncu_full_cfg3.log 2>&1
echo done > $O/done
