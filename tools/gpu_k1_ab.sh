#!/bin/bash
# Dev tool (GPU box): cfg3 nrhs=1 A/B of the default build against a variant (VAR).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-k1ab}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "matvec or k1" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1300 python tools/build_time.py 256 --save /tmp/cfg3_256.hvfm > $O/build.log 2>&1
timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --fhat /tmp/cfg3_256.hvfm --no-cpu-baseline > $O/bench_default.log 2>&1
VF_LIB=paper_2209_07632_b200/build/var_${VAR:-nocsrvec}.so timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --fhat /tmp/cfg3_256.hvfm --no-cpu-baseline --no-parity > $O/bench_var.log 2>&1
timeout 300 python bench.py --workload cfg3 --nrhs 128 --steps 10 --warmup 3 --fhat /tmp/cfg3_256.hvfm --no-cpu-baseline --no-parity > $O/bench_k128.log 2>&1
timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 --fhat /tmp/cfg3_256.hvfm --no-cpu-baseline > $O/bench_cfg5.log 2>&1
echo done > $O/done
