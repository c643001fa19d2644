F=/tmp/cfg3_p1.hvfm
python bench.py --workload cfg3 --nrhs 1 --steps 20 --warmup 3 --no-cpu-baseline --fhat $F > gpurun_out/cs_1.log 2>&1
for K in 2 4 8; do
  python bench.py --workload cfg3 --nrhs $K --steps 20 --warmup 3 --no-cpu-baseline --fhat $F > gpurun_out/cs_$K.log 2>&1
done
