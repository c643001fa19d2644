#!/bin/bash
# Dev tool (GPU box): final cfg2 evidence (bench lines, ncu launch list, full capture, trace).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-cfg2final}
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 400 python bench.py --steps 100 --warmup 5 > $O/bench_cfg2.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 --dtype f32 --no-cpu-baseline > $O/bench_cfg2_f32.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_cfg2_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/ncu_launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch_cfg2.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:res_kernel -s 2 -c 1 -o $O/res_full_cfg2 python tools/solve_once.py > $O/ncu_full_cfg2.log 2>&1
timeout 200 python tools/trace.py $O/trace_cfg2.bin --run > $O/trace_cfg2.txt 2>&1
echo done > $O/done
