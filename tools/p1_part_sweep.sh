set -x
F=/tmp/cfg3_p1.hvfm
python bench.py --workload cfg3 --steps 100 --warmup 5 --no-cpu-baseline --fhat $F > gpurun_out/p1_2048a.log 2>&1
for P in 512 1024 4096 2048 256; do
  VF_P1_PART=$P python bench.py --workload cfg3 --steps 100 --warmup 5 --no-cpu-baseline --fhat $F > gpurun_out/p1_$P.log 2>&1
done
for f in gpurun_out/p1_*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])"; done
