#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2; do
  r=$(EMRKC_PROBE_FAST_ONLY=1 timeout 300 python tools/probe.py hh3d_128x128x128 hh3d_256x256x128 hh3d_512x512x256 2>&1 | awk '{print $2, $8, $9}' | tr '\n' ' ')
  echo "rep=$rep :: $r"
done
