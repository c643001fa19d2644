#!/bin/bash
# Dev tool (runs on the GPU box): build/load the cfg3 F-hat once, then the
# cfg3 / cfg5 bench lines, the ncu launch list and one full ncu capture.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-cfg3}
mkdir -p $O
F=/tmp/cfg3_{n}.hvfm
timeout 1500 python tools/build_time.py 256 --save /tmp/cfg3_256.hvfm > $O/build.log 2>&1 || true
timeout 900 python bench.py --workload cfg3 --nrhs 1 --steps 30 --warmup 5 --fhat $F > $O/bench_cfg3_k1.log 2>&1
timeout 900 python bench.py --workload cfg3 --nrhs 128 --steps 10 --warmup 3 --fhat $F --no-cpu-baseline --no-parity > $O/bench_cfg3_k128.log 2>&1
timeout 900 python bench.py --workload cfg5 --steps 5 --warmup 3 --fhat $F > $O/bench_cfg5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/ncu_launches_cfg3_k1.csv python bench.py --workload cfg3 --nrhs 1 --steps 3 --warmup 3 --fhat $F --no-cpu-baseline --no-parity > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 3 -c 1 -o $O/hot_cfg3_k1 python tools/mv_once.py 256 1 /tmp/cfg3_256.hvfm > $O/ncu_full.log 2>&1
echo done > $O/done
