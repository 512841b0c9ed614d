#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for pipe in 1 0; do
  r=$(EMRKC_PIPE=$pipe EMRKC_PROBE_FAST_ONLY=1 timeout 300 python tools/probe.py hh3d_512x512x256 hh3d_sweep_200 hh3d_sweep_100 hh3d_128x128x128 2>&1 | awk '{print $2, $5, $8, $9}' | tr '\n' ' ')
  echo "pipe=$pipe :: $r"
done
