#!/bin/bash
# round 2, session 36: tools/stream_probe -- the HBM rate the nrhs = 1 row kernel's
# access pattern allows (rounds in flight per warp, with / without dependent gathers)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s36; mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 600 tools/stream_probe > $O/stream_probe.txt 2>&1
timeout 600 tools/stream_probe 131072 19 >> $O/stream_probe.txt 2>&1
timeout 600 tools/stream_probe 32768 76 > $O/stream_probe_long_rows.txt 2>&1
echo done > $O/done
