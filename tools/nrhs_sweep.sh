# cfg3 F-hat (tol 1e-5) applied to nrhs = 1..256 columns; F-hat cached in /tmp
F=${1:-/tmp/cfg3_p1.hvfm}
for K in 1 2 4 8 16 32 64 128 256; do
  python bench.py --workload cfg3 --nrhs $K --steps 20 --warmup 3 --no-cpu-baseline --fhat $F > gpurun_out/nrhs_$K.log 2>&1
done
