#!/bin/bash
# A/B of two libraries through tools/probe.py: tools/ab_lib.sh <libA> <libB> workloads...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
la=$1; lb=$2; shift 2
for rep in 1 2; do
for wl in "$@"; do
  for l in $la $lb; do
    echo "rep=$rep $l $(EMRKC_LIB=$l EMRKC_PROBE_FAST_ONLY=1 timeout 300 python tools/probe.py $wl 2>&1 | tail -1 | cut -c1-110)"
  done
done
done
