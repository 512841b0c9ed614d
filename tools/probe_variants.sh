#!/bin/bash
# Times the emRKC step for each library variant in build_var/, pipe on/off, zc.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for lib in build_var/*.so; do
  for pipe in 1 0; do
    for zc in 8 16 32; do
      echo "== $lib pipe=$pipe zc=$zc"
      EMRKC_PIPE=$pipe EMRKC_ZC=$zc EMRKC_LIB=$PWD/$lib EMRKC_PROBE_FAST_ONLY=1 timeout 300 python tools/probe.py hh3d_128x128x128 2>&1 | tail -1
    done
  done
done
