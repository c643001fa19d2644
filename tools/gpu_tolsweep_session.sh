#!/bin/bash
# Dev tool (GPU box): configs[2] tolerance sweep -- build F-hat at each tol
# (untimed, cached under /tmp) and run the cfg3 nrhs = 1 bench line on it;
# then A/B of the x-gather load path on the tol 1e-5 ... (uses whatever is cached).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-tolsweep}
mkdir -p $O
for tol in ${TOLS:-1e-7 1e-3}; do
  timeout ${BUILD_LIMIT:-1500} python tools/build_time.py 256 --tol $tol --save /tmp/cfg3_256_$tol.hvfm > $O/build_$tol.log 2>&1
  if [ -f /tmp/cfg3_256_$tol.hvfm ]; then
    timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --tol $tol --fhat /tmp/cfg3_256_$tol.hvfm --no-cpu-baseline > $O/bench_cfg3_k1_$tol.log 2>&1
    export VF_LIB=paper_2209_07632_b200/build/var_ldg.so
    timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --tol $tol --fhat /tmp/cfg3_256_$tol.hvfm --no-cpu-baseline --no-parity > $O/bench_cfg3_k1_${tol}_ldg.log 2>&1
    unset VF_LIB
  fi
done
echo done > $O/done
