#!/bin/bash
# Dev tool (GPU box): cfg3 FP32 nrhs=1 A/B (default vs VARS).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-f32k1}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "f32" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1300 python bench.py --workload cfg3 --dtype f32 --nrhs 1 --steps 300 --warmup 5 --fhat /tmp/cfg3_f32.hvfm --no-cpu-baseline > $O/bench_default.log 2>&1
for v in $VARS; do
  VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 python bench.py --workload cfg3 --dtype f32 --nrhs 1 --steps 300 --warmup 5 --fhat /tmp/cfg3_f32.hvfm --no-cpu-baseline --no-parity > $O/bench_$v.log 2>&1
done
echo done > $O/done
