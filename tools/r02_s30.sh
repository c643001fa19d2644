#!/bin/bash
# round 2, session 30: (1) compact 16-B run descriptors in the nrhs = 1 row
# kernel (SegC) — A/B against the previous build (libvf_head.so) on
# configs[2], alternating; (2) FP32 wide batches on DMMA (bt_kernel<float>)
# vs the tcgen05 3xTF32 kernels; GPU tests of both
cd $GRAFT_REPO_ROOT
O=gpurun_out/s30; mkdir -p $O
F=/tmp/cfg3.hvfm
F32=/tmp/cfg3_f32.hvfm
P=paper_2209_07632_b200
nvidia-smi > $O/nvidia_smi.txt 2>&1
( time timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q ) > $O/pytest_tiles.log 2>&1; echo "rc $?" >> $O/pytest_tiles.log
[ -f $F ] || ( time timeout 1500 python tools/mv_once.py 256 1 $F ) > $O/build.log 2>&1
B="python bench.py --fhat $F --no-cpu-baseline --batched 0 --steps 200"
for i in 1 2; do
  VF_LIB=$P/libvf_head.so timeout 600 $B > $O/bench_head_$i.json 2> $O/bench_head_$i.err
  timeout 600 $B > $O/bench_segc_$i.json 2> $O/bench_segc_$i.err
done
timeout 600 python bench.py --fhat $F --no-cpu-baseline --batched 0 --nrhs 128 --steps 10 > $O/bench_k128.json 2> $O/bench_k128.err
B32="python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --nrhs 128 --batched 0 --steps 10"
( time timeout 1500 $B32 ) > $O/bench_f32_k128_dmma.json 2> $O/bench_f32_k128_dmma.err
VF_TC2=1 timeout 600 $B32 > $O/bench_f32_k128_tc2.json 2> $O/bench_f32_k128_tc2.err
timeout 600 python bench.py --fhat $F32 --dtype f32 --no-cpu-baseline --nrhs 64 --batched 0 --steps 10 > $O/bench_f32_k64_dmma.json 2> $O/bench_f32_k64_dmma.err
( time timeout 1500 python -m pytest tests/test_gpu_k1p.py tests/test_gpu_rows.py tests/test_gpu_parity.py -x -q ) > $O/pytest.log 2>&1; echo "rc $?" >> $O/pytest.log
timeout 900 python bench.py --fhat $F --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
echo done > $O/done
