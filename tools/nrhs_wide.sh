F=/tmp/cfg3_p1.hvfm
for K in 100 150 128 4 1; do
  python bench.py --workload cfg3 --nrhs $K --steps 10 --warmup 3 --no-cpu-baseline --fhat $F > gpurun_out/ch2_$K.log 2>&1
done
