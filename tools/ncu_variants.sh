#!/bin/bash
# ncu --set full of the node kernel for two library variants (one short probe each).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # tag lib pipe zc
  CMD="python tools/probe.py hh3d_128x128x128"
  EMRKC_PIPE=$3 EMRKC_ZC=$4 EMRKC_LIB=$PWD/$2 EMRKC_PROBE_FAST_ONLY=1 $CMD > gpurun_out/plain_$1.log 2>&1 && \
  EMRKC_PIPE=$3 EMRKC_ZC=$4 EMRKC_LIB=$PWD/$2 EMRKC_PROBE_FAST_ONLY=1 ncu --set full --clock-control none --import-source on \
     -k regex:'k_node' -s 5 -c 1 -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
}
run pipe build_var/lib_nb6_pb6.so 1 8
run march build_var/lib_nb8_pb8.so 0 16
