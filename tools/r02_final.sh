#!/bin/bash
# round 2, final evidence: GPU suite + smoke, the driver's default bench line
# (builds configs[2]), reference arm, ncu launch list of the default command,
# full capture of the dominant kernel, batched capture
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
F=/tmp/cfg3.hvfm
nvidia-smi > $O/nvidia_smi.txt 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
( time timeout 2400 python bench.py --fhat $F ) > $O/bench_default.json 2> $O/bench_default.err
( time timeout 900 python bench.py --impl reference --steps 5 --warmup 3 ) > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 5 --warmup 3 > $O/ncu_launches.log 2>&1
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1 python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
timeout 300 python tools/mv_once.py 256 128 $F > $O/mv128_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_kernel -s 1 -c 1 -o $O/bt python tools/mv_once.py 256 128 $F > $O/ncu_bt.log 2>&1
echo done > $O/done
