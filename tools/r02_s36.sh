#!/bin/bash
# round 2, session 36: tools/stream_probe -- the HBM rate the nrhs = 1 row kernel's
# access pattern allows (rounds in flight per warp, with / without dependent gathers);
# two register rounds in flight (VF_K1_PFD=2) again, now on the shuffle-free fetch
# (fewer live registers): 4 CTAs / 64 registers with and without the queue code,
# 3 CTAs / 74 registers without spills
cd $GRAFT_REPO_ROOT
O=gpurun_out/s36; mkdir -p $O
F=/tmp/cfg3.hvfm
P=paper_2209_07632_b200
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 600 tools/stream_probe > $O/stream_probe.txt 2>&1
timeout 600 tools/stream_probe 32768 76 > $O/stream_probe_long_rows.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
for i in 1 2; do
  timeout 600 $B > $O/bench_default_$i.json 2> $O/bench_default_$i.err
  for v in pfd2 pfd2ns pfd2c3; do
    VF_LIB=$P/build/var_$v.so timeout 600 $B > $O/bench_${v}_$i.json 2> $O/bench_${v}_$i.err
  done
done
VF_LIB=$P/build/var_pfd2c3.so timeout 900 python -m pytest tests/test_gpu_k1p.py -x -q -k "forced_layouts or smq" > $O/pytest_pfd2c3.log 2>&1; echo "rc $?" >> $O/pytest_pfd2c3.log
echo done > $O/done
