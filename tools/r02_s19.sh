#!/bin/bash
# round 2, session 19: column-split solves (tests + cfg3 timing), resident
# phase-2 copies (tests + cfg2 bench A/B + phase trace)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s19; mkdir -p $O
F=/tmp/cfg3.hvfm
ls -la $F > $O/cache.txt 2>&1
( time timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "column_split_solves or phase2_copies or resident_and_streaming or radiosity or thermal" ) > $O/pytest_new.log 2>&1; echo "rc $?" >> $O/pytest_new.log
( time timeout 900 python -m pytest tests/test_gpu_k1p.py -x -q ) > $O/pytest_k1p.log 2>&1; echo "rc $?" >> $O/pytest_k1p.log
for c in 4 2 1; do
  VF_RES_P2COPIES=$c timeout 400 python bench.py --workload cfg2 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_cfg2_c$c.json 2> $O/bench_cfg2_c$c.err
done
timeout 400 python bench.py --workload cfg2 --steps 100 --warmup 5 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 200 python tools/trace.py /tmp/trace_cfg2.bin --run > $O/trace_cfg2.txt 2>&1
VF_RES_P2COPIES=1 timeout 200 python tools/trace.py /tmp/trace_cfg2_c1.bin --run > $O/trace_cfg2_c1.txt 2>&1
[ -f $F ] && timeout 1200 python tools/solve_cols.py $F 1,2,4,8 > $O/solve_cols.txt 2>&1
echo done > $O/done
