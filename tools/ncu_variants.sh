#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
EMRKC_PROBE_FAST_ONLY=1 python tools/probe.py hh3d_128x128x128 hh3d_512x512x256 2>&1 | tail -2
CMD="python tools/probe.py hh3d_128x128x128"
EMRKC_PROBE_FAST_ONLY=1 $CMD > gpurun_out/plain_pipe.log 2>&1 && \
EMRKC_PROBE_FAST_ONLY=1 ncu --set full --clock-control none --import-source on -k regex:'k_node' -s 5 -c 1 -o gpurun_out/prof_pipe2 $CMD > gpurun_out/ncu_pipe2.log 2>&1
echo "ncu rc=$?"
