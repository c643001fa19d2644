#!/bin/bash
# Dev tool (runs on the GPU box): gpu tests, smoke, the default bench line
# (BASELINE configs[1]), its ncu launch list and one full capture of the
# dominant kernel.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-cfg2}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > $O/bench.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --dtype f32 --no-cpu-baseline > $O/bench_f32.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/ncu_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:res_kernel -s 2 -c 1 -o $O/res_full python tools/solve_once.py > $O/ncu_full.log 2>&1
timeout 300 python tools/trace.py $O/trace.bin --run > $O/trace.txt 2>&1
echo done > $O/done
