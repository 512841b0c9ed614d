#!/bin/bash
# A/B of the temporally blocked inner stages (EMRKC_TB) through tools/probe.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for wl in "$@"; do
  for tb in 0 1; do
    echo "TB=$tb $(EMRKC_TB=$tb EMRKC_PROBE_FAST_ONLY=1 timeout 300 python tools/probe.py $wl 2>&1 | tail -1)"
  done
done
