#!/bin/bash
# round 2, session 37: rehearsal of the driver's round-end commands on the final
# build (no cached F-hat: bench.py builds configs[2] itself)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s37; mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
( time timeout 600 python bench.py --impl reference ) > $O/bench_reference.json 2> $O/bench_reference.err
( time timeout 2400 python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
echo done > $O/done
