#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s9; mkdir -p $O
timeout 120 ./tools/tc_probe > $O/tc_probe.log 2>&1; echo "rc $?" >> $O/tc_probe.log
