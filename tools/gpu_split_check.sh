#!/bin/bash
# Dev tool (GPU box): resident-kernel cluster split A/B -- parity tests, phase
# traces and the default bench line with VF_RES_SPLIT=1 (default) and 0.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-split}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
for sp in 1 0; do
  VF_RES_SPLIT=$sp timeout 200 python tools/trace.py $O/trace_$sp.bin --run > $O/trace_split$sp.txt 2>&1
  VF_RES_SPLIT=$sp timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_split$sp.log 2>&1
done
echo done > $O/done
