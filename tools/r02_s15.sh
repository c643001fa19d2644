#!/bin/bash
# round 2, session 15: k1p_kernel (pipelined nrhs = 1) parity + cfg3 A/B vs the
# row kernel, ring depth / CTA variants, ncu capture of k1p
cd $GRAFT_REPO_ROOT
O=gpurun_out/s15; mkdir -p $O
F=/tmp/cfg3.hvfm
ls -la $F > $O/cache.txt 2>&1
nvidia-smi > $O/nvidia_smi.txt 2>&1
( time timeout 900 python -m pytest tests/test_gpu_k1p.py -x -q ) > $O/pytest_k1p.log 2>&1; echo "rc $?" >> $O/pytest_k1p.log
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
VF_K1_KERNEL=rows timeout 600 $B > $O/bench_rows.json 2> $O/bench_rows.err
VF_K1_KERNEL=pipe timeout 600 $B > $O/bench_pipe.json 2> $O/bench_pipe.err
for v in d3 d6c3 d8c2; do
  VF_K1_KERNEL=pipe VF_LIB=paper_2209_07632_b200/build/var_$v.so timeout 600 $B > $O/bench_$v.json 2> $O/bench_$v.err
done
VF_K1_KERNEL=pipe timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_pipe.log 2>&1 && \
VF_K1_KERNEL=pipe timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1p_kernel -s 1 -c 1 -o $O/k1p python tools/mv_once.py 256 1 $F > $O/ncu_k1p.log 2>&1
( time timeout 1800 python -m pytest tests -m gpu -x -q ) > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
echo done > $O/done
