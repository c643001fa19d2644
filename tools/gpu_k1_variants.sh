#!/bin/bash
# Dev tool (GPU box): cfg3 nrhs=1 bench for the default build and variants (VARS).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-k1var}
mkdir -p $O
timeout 1300 python tools/build_time.py 256 --save /tmp/cfg3_256.hvfm > $O/build.log 2>&1
timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --fhat /tmp/cfg3_256.hvfm --no-cpu-baseline --no-parity > $O/bench_default.log 2>&1
for v in $VARS; do
  VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --fhat /tmp/cfg3_256.hvfm --no-cpu-baseline --no-parity > $O/bench_$v.log 2>&1
done
echo done > $O/done
