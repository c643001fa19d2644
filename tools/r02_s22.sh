#!/bin/bash
# round 2, session 22: per-row contiguous 16-bit layout (dense/U runs copied next
# to the interleaved CSR pieces) A/B; bt_kernel half-tile DMMAs A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s22; mkdir -p $O
F=/tmp/cfg3.hvfm
ls -la $F > $O/cache.txt 2>&1
( time timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_k1p.py tests/test_gpu_tiles.py -x -q -k "k1 or matvec or tiles or column or timestep or k1p" ) > $O/pytest_a.log 2>&1; echo "rc $?" >> $O/pytest_a.log
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
timeout 600 $B > $O/bench_pack.json 2> $O/bench_pack.err
VF_K1_PACK=0 timeout 600 $B > $O/bench_nopack.json 2> $O/bench_nopack.err
VF_K1_ILV=0 timeout 600 $B > $O/bench_pack_plain.json 2> $O/bench_pack_plain.err
timeout 600 $B > $O/bench_pack2.json 2> $O/bench_pack2.err
for k in 128 64; do
  timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k$k.json 2> $O/bench_k$k.err
  VF_LIB=paper_2209_07632_b200/build/var_nohalf.so timeout 600 python bench.py --fhat $F --no-cpu-baseline --nrhs $k --batched 0 --steps 10 > $O/bench_k${k}_nohalf.json 2> $O/bench_k${k}_nohalf.err
done
timeout 300 python tools/trace_matvec.py 256 1 $F > $O/trace.txt 2>&1
timeout 300 python tools/mv_once.py 256 1 $F > $O/mv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 1 -c 1 -o $O/hot python tools/mv_once.py 256 1 $F > $O/ncu_hot.log 2>&1
echo done > $O/done
