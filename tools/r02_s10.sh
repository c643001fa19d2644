#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s10; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q -k f32 > $O/pytest_tc.log 2>&1; echo "rc $?" >> $O/pytest_tc.log
