#!/bin/bash
# Dev tool (GPU box): parity tests + cfg3 nrhs=128 on the cached F-hat with the
# wide per-row path (default) vs the row-group path (VF_WIDE=0).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-wide}
mkdir -p $O
ls -la /tmp/cfg3_256.hvfm > $O/ls.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 1500 python bench.py --workload cfg3 --nrhs 128 --steps 10 --warmup 3 --fhat /tmp/cfg3_256.hvfm --no-cpu-baseline --no-parity > $O/bench_cfg3_k128.log 2>&1
timeout 600 python bench.py --workload cfg3 --nrhs 128 --steps 5 --warmup 2 --fhat /tmp/cfg3_256.hvfm --no-cpu-baseline > $O/bench_cfg3_k128_parity.log 2>&1
timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 --fhat /tmp/cfg3_256.hvfm > $O/bench_cfg5.log 2>&1
echo done > $O/done
