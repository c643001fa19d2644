#!/bin/bash
# round 2, session 2: stream kernel tests, GPU suite, default bench with stats
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/s2/pytest_stream.log 2>&1; echo "rc $?" >> gpurun_out/s2/pytest_stream.log
if grep -q "rc 0" gpurun_out/s2/pytest_stream.log; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/s2/pytest_gpu.log
  VF_LAYOUT_STATS=1 VF_BUILD_PROFILE=1 timeout 1800 python bench.py --fhat /tmp/cfg3_{n}_{tol}_{dtype}.hvfm --no-cpu-baseline > gpurun_out/s2/bench.json 2> gpurun_out/s2/bench.err; echo "bench rc $?" >> gpurun_out/s2/bench.err
  VF_NO_STREAM=1 timeout 900 python bench.py --fhat /tmp/cfg3_{n}_{tol}_{dtype}.hvfm --no-cpu-baseline --batched 0 > gpurun_out/s2/bench_nostream.json 2> gpurun_out/s2/bench_nostream.err
fi
