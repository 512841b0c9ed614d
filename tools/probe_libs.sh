#!/bin/bash
# probe.py over library variants: "name=path" pairs in LIBS (default lib: "base=").
cd "${GRAFT_REPO_ROOT:-/root/repo}"
W=${W:-"hh3d_128x128x128 hh3d_256x256x128 hh3d_512x512x256 hh2d_256x256 hh3d_sweep_100"}
for rep in 1 2; do
  for lv in $LIBS; do
    n=${lv%%=*}; l=${lv#*=}
    r=$(EMRKC_LIB=$l EMRKC_PROBE_FAST_ONLY=1 timeout 300 python tools/probe.py $W 2>&1 | awk '{print $2, $9}' | tr '\n' ' ')
    echo "rep=$rep $n $EMRKC_PIPE :: $r"
  done
done
