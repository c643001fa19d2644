#!/bin/bash
# compute-sanitizer racecheck on a small case launching every kernel family (one tool per call)
cd $GRAFT_REPO_ROOT
O=gpurun_out/san; mkdir -p $O
timeout 600 python tools/sanitize_case.py > $O/plain.log 2>&1; echo "rc $?" >> $O/plain.log
grep -q "sanitize case ok" $O/plain.log || exit 1
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_case.py > $O/racecheck.log 2>&1; echo "rc $?" >> $O/racecheck.log
