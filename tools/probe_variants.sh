#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for lib in build_var/*.so; do
  for zc in 8 16 32; do
    r=$(EMRKC_PIPE=1 EMRKC_ZC=$zc EMRKC_LIB=$PWD/$lib EMRKC_PROBE_FAST_ONLY=1 timeout 300 python tools/probe.py hh3d_128x128x128 hh3d_512x512x256 2>&1 | awk '{print $2, $8, $9}' | tr '\n' ' ')
    echo "$lib zc=$zc :: $r"
  done
done
