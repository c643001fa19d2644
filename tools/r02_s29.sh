#!/bin/bash
# round 2, session 29: the new GPU tests (default row kernel under forced
# layouts; configs[2] recipe at 64^2 cells vs the exact F)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s29; mkdir -p $O
( time timeout 1500 python -m pytest tests/test_gpu_k1p.py tests/test_gpu_parity.py -q -k "default_row_kernel or terrain64 or column_split or phase2_copies" ) > $O/pytest_new.log 2>&1; echo "rc $?" >> $O/pytest_new.log
echo done > $O/done
