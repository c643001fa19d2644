#!/bin/bash
# round 2, session 33: per-SM row queues of the nrhs = 1 matvec (VF_K1_SMQ) on
# configs[2]: the kernel without the queue code (var_nosmq), the new build with
# the global queue (SMQ=0), SMQ=1 at pool thresholds 1 / 2 / 4 / none, and with
# T rows through L1 (var_tl1); the nrhs = 1 GPU tests on the new build; ncu of
# the best setting
cd $GRAFT_REPO_ROOT
O=gpurun_out/s33; mkdir -p $O
F=/tmp/cfg3.hvfm
P=paper_2209_07632_b200
nvidia-smi > $O/nvidia_smi.txt 2>&1
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
for i in 1 2; do
  VF_LIB=$P/build/var_nosmq.so timeout 600 $B > $O/bench_nosmq_$i.json 2> $O/bench_nosmq_$i.err
  VF_K1_SMQ=0 timeout 600 $B > $O/bench_smq0_$i.json 2> $O/bench_smq0_$i.err
  for thr in 1 2 4 1e9; do
    VF_K1_SMQ=1 VF_K1_SMQ_THR=$thr VF_LAYOUT_DEBUG=1 timeout 600 $B > $O/bench_smq1_thr${thr}_$i.json 2> $O/bench_smq1_thr${thr}_$i.err
    VF_LIB=$P/build/var_tl1.so VF_K1_SMQ=1 VF_K1_SMQ_THR=$thr timeout 600 $B > $O/bench_smq1_tl1_thr${thr}_$i.json 2> $O/bench_smq1_tl1_thr${thr}_$i.err
  done
  VF_LIB=$P/build/var_tl1.so VF_K1_SMQ=1 VF_K1_SMQ_THR=2 VF_K1_OVL=1 timeout 600 $B > $O/bench_smq1_tl1_ovl_$i.json 2> $O/bench_smq1_tl1_ovl_$i.err
done
( time timeout 1500 python -m pytest tests/test_gpu_k1p.py -x -q ) > $O/pytest_k1p.log 2>&1; echo "rc $?" >> $O/pytest_k1p.log
VF_K1_SMQ=1 timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace_smq1.txt 2>&1
VF_LIB=$P/build/var_tl1.so VF_K1_SMQ=1 timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
VF_LIB=$P/build/var_tl1.so VF_K1_SMQ=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1_smq_tl1 python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
VF_K1_SMQ=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot_k1_smq python tools/mv_once.py 256 1 $F > $O/ncu_hot2.log 2>&1
echo done > $O/done
