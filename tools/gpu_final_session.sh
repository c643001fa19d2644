#!/bin/bash
# Dev tool (GPU box): the round's final evidence in one call -- gpu tests,
# smoke, cfg2 bench lines (f64, f32, reference arm), ncu launch list + full
# capture of res_kernel, then the cfg3 build and its nrhs=1 / 128 and cfg5
# lines with ncu launch list + full capture of the nrhs=1 hot kernel.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-final}
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 400 python bench.py --steps 100 --warmup 5 > $O/bench_cfg2.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 --dtype f32 --no-cpu-baseline > $O/bench_cfg2_f32.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_cfg2_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/ncu_launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch_cfg2.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:res_kernel -s 2 -c 1 -o $O/res_full_cfg2 python tools/solve_once.py > $O/ncu_full_cfg2.log 2>&1
timeout 200 python tools/trace.py $O/trace_cfg2.bin --run > $O/trace_cfg2.txt 2>&1
timeout 1300 python tools/build_time.py 256 --save /tmp/cfg3_256.hvfm > $O/build_cfg3.log 2>&1
F=/tmp/cfg3_256.hvfm
timeout 600 python bench.py --workload cfg3 --nrhs 1 --steps 300 --warmup 5 --fhat $F > $O/bench_cfg3_k1.log 2>&1
timeout 300 python bench.py --workload cfg3 --nrhs 128 --steps 10 --warmup 3 --fhat $F --no-cpu-baseline --no-parity > $O/bench_cfg3_k128.log 2>&1
timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 --fhat $F > $O/bench_cfg5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/ncu_launches_cfg3_k1.csv python bench.py --workload cfg3 --nrhs 1 --steps 3 --warmup 3 --fhat $F --no-cpu-baseline --no-parity > $O/ncu_launch_cfg3.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:hot_kernel -s 3 -c 1 -o $O/hot_full_cfg3_k1 python tools/mv_once.py 256 1 $F > $O/ncu_full_cfg3.log 2>&1
echo done > $O/done
