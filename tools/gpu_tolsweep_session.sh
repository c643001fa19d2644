#!/bin/bash
# Dev tool (GPU box): configs[2] tolerance sweep -- build F-hat at each tol
# (untimed, cached under /tmp) and run the cfg3 nrhs = 1 bench line on it.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-tolsweep}
mkdir -p $O
for tol in ${TOLS:-1e-3 1e-7}; do
  timeout 2400 python tools/build_time.py 256 --tol $tol --save /tmp/cfg3_256_$tol.hvfm > $O/build_$tol.log 2>&1
  timeout 900 python bench.py --workload cfg3 --nrhs 1 --steps 100 --warmup 5 --tol $tol --fhat /tmp/cfg3_256_$tol.hvfm --no-cpu-baseline > $O/bench_cfg3_k1_$tol.log 2>&1
done
echo done > $O/done
