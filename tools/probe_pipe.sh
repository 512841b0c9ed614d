#!/bin/bash
# Device ms/step of each staged-kernel family (EMRKC_PIPE) on the bench grids.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
W=${W:-"hh3d_128x128x128 hh3d_256x256x128 hh3d_512x512x256 hh2d_256x256 hh3d_sweep_100"}
for rep in 1 2; do
  for pp in ${PIPES:-1 3}; do
    r=$(EMRKC_PIPE=$pp EMRKC_PROBE_FAST_ONLY=1 timeout 300 python tools/probe.py $W 2>&1 | awk '{print $2, $4, $8, $9}' | tr '\n' ' ')
    echo "rep=$rep pipe=$pp :: $r"
  done
done
