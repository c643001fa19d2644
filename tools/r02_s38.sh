#!/bin/bash
# round 2, session 38: stream_probe with padded rounds (extra instructions per
# lane and round), to see at what instruction count the access pattern leaves the HBM roof
cd $GRAFT_REPO_ROOT
O=gpurun_out/s38; mkdir -p $O
timeout 600 tools/stream_probe > $O/stream_probe_pad.txt 2>&1
echo done > $O/done
