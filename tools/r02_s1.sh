#!/bin/bash
# round 2, session 1: GPU tests, default bench line, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1/gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s1/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/s1/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/s1/bench.json 2> gpurun_out/s1/bench.err; echo "bench rc $?" >> gpurun_out/s1/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/s1/ref.json 2> gpurun_out/s1/ref.err
